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
#include <cstdio>
#include <cstdlib>

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

// X(r, c) = uniform[-1, 1) from the hash of (seed, r, c), r < rows, c < cols (ld ldx)
__global__ void __launch_bounds__(256) fill_uniform_kernel(double* X, int ldx, int rows, int cols,
                                                           unsigned long long seed) {
  const long long tot = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % rows), c = int(e / rows);
    X[r + (long long)c * ldx] = hash_uniform((seed << 40) ^ ((unsigned long long)r * 0x100000001B3ull + c));
  }
}

cudaError_t launch_fill_uniform(double* X, int ldx, int rows, int cols, unsigned long long seed, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const long long tot = (long long)rows * cols;
  fill_uniform_kernel<<<unsigned(std::min<long long>((tot + 255) / 256, 1184)), 256, 0, st>>>(X, ldx, rows, cols, seed);
  return cudaGetLastError();
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
// Q = H_0 ... H_{n-1} [I; 0] (m x n), LAPACK dgeqr2 / dorg2r conventions
// (H = I - tau v v^T, v_c = 1, beta = -sign(alpha) ||x||; Q formed in place over
// the reflectors). One thread-block cluster of C CTAs per matrix: CTA r owns rows
// [r R, (r + 1) R) and keeps them in shared memory (SM) or works on them in place in
// global memory (large matrices). A column step is two phases: warp 0 forms the
// reflector (norm by a warp reduction, scaling by all lanes); then groups of 8
// lanes own the trailing columns (dot product over the rows, a 3-step shuffle
// reduction, the update of the same rows). With C > 1 the partial norms and dot
// products are summed over the cluster through DSMEM in rank order, so every CTA
// forms bit-identical reflectors; reduction slots alternate by column parity. The
// reflectors are applied to the p probe columns too: their rows n..m-1 then hold
// (I - Q Q^T) y, the randomized range finder's a-posteriori estimate (Halko,
// Martinsson & Tropp 2011, Sec. 4.3). stat[1] = max_probe |(I - Q Q^T) y| / scale,
// stat[0] = #{|R_ii| > eps scale}, relative to the box operator's scale
// max_i |S_ii| sqrt(k / 3) (the expected norm of S applied to a k-vector of
// uniform[-1, 1] entries; S is diagonally dominant).
constexpr int QR_THREADS = 256, QR_WARPS = QR_THREADS / 32, QR_MAXC = 16, QR_MAXN = 256;
constexpr int QR_GL = 8, QR_NG = QR_THREADS / QR_GL;  // lanes per column group, column groups

struct QrShared {
  double nrm[QR_MAXN];         // PIV: trailing column norms^2 (cluster sums)
  double wsum[QR_MAXN];        // cluster-summed dot products of the current step
  int jmax;                    // PIV: pivot column of this step
  double a[2][2];              // [parity] partial sum of squares, alpha (the row owner's)
  double w[2][QR_MAXN + 8];    // [parity] partial dot products
  double tau[QR_MAXN], rdiag[QR_MAXN];
  double red[QR_WARPS];
};

// PIV: Householder QR with column pivoting (largest remaining column norm first,
// lowest index on ties; LAPACK dgeqp3's rule with norms recomputed each step) --
// the rank-revealing QR of the compressed engine's basis selection (hbs.cu); stat[0]
// then counts |R_ii| > eps |R_00| (QrDesc::S == nullptr).
template <bool CL, bool SM, bool PIV = false>
__global__ void __launch_bounds__(QR_THREADS) hqr_kernel(const QrDesc* __restrict__ descs, const double* eps_ptr,
                                                         int C) {
  extern __shared__ __align__(16) double qdyn[];
  __shared__ QrShared sh;
  const int rank = CL ? int(cg::this_cluster().block_rank()) : 0;
  auto csync = [] {
    if constexpr (CL) cg::this_cluster().sync();
  };
  auto remote = [&](double* p, int q) -> double {
    if constexpr (CL) return *cg::this_cluster().map_shared_rank(p, q);
    else return *p;
  };
  const QrDesc d = descs[blockIdx.x / C];
  const int m = d.m, n = d.n, nc = d.n + d.p;
  const int R = (m + C - 1) / C, r0 = rank * R, r1 = min(m, r0 + R), nr = max(r1 - r0, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gl = tid & (QR_GL - 1), grp = tid / QR_GL;
  const long long ld = SM ? (nr | 1) : d.ldy;
  double* Y = SM ? qdyn : d.Y + r0;  // local rows, column-major
  if constexpr (SM) {
    for (int j = 0; j < nc; ++j)
      for (int i = tid; i < nr; i += QR_THREADS) Y[i + j * ld] = d.Y[r0 + i + (long long)j * d.ldy];
    __syncthreads();
  }
  // trailing-column phase: every column j in [j0, j1) -> dot with the reflector in
  // column c (rows >= c; v_c = 1), summed over the cluster, and y_j -= tau (v . y_j) v
  auto apply_reflector = [&](int c, int j0, int j1, int par) {
    const double tc = sh.tau[c];
    const double* yc = Y + c * ld;
    const bool own_row = c >= r0 && c < r1;
    const int lv = max(c - r0, 0);
    // the group's dot product v . y_j (every lane of the warp must call it: it shuffles)
    auto partial_dot = [&](int j, bool valid) {
      double dot = 0.0;
      if (valid) {
        const double* yj = Y + j * ld;
        double s0 = 0.0, s1 = 0.0;
        int i = lv + gl;
        if (own_row && gl == 0) {
          s0 = yj[lv];
          i += QR_GL;
        }
        for (; i + QR_GL < nr; i += 2 * QR_GL) {
          s0 = fma(yc[i], yj[i], s0);
          s1 = fma(yc[i + QR_GL], yj[i + QR_GL], s1);
        }
        if (i < nr) s0 = fma(yc[i], yj[i], s0);
        dot = s0 + s1;
      }
#pragma unroll
      for (int o = QR_GL / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      return dot;
    };
    auto update = [&](int j, double dot) {
      double* yj = Y + j * ld;
      const double f = tc * dot;
      int i = lv + gl;
      if (own_row && gl == 0) {
        yj[lv] -= f;
        i += QR_GL;
      }
      for (; i < nr; i += QR_GL) yj[i] = fma(-f, yc[i], yj[i]);
    };
    if constexpr (CL) {
      // every trailing column's partial dot (slots indexed by column: one barrier), then
      // the cluster sums and the updates
      for (int jb = j0; jb < j1; jb += QR_NG) {
        const int j = jb + grp;
        const double dot = partial_dot(j, j < j1);
        if (j < j1 && gl == 0) sh.w[par][j] = dot;
      }
      csync();
      // one thread per column sums the C partials (independent DSMEM loads, in flight
      // together), rank order
      for (int j = j0 + tid; j < j1; j += QR_THREADS) {
        double t = 0.0;
        for (int q = 0; q < C; ++q) t += remote(&sh.w[par][j], q);
        sh.wsum[j] = t;
      }
      __syncthreads();
      if (tc != 0.0)
        for (int jb = j0; jb < j1; jb += QR_NG) {
          const int j = jb + grp;
          if (j < j1) update(j, sh.wsum[j]);
        }
    } else {
      if (tc != 0.0)
        for (int jb = j0; jb < j1; jb += QR_NG) {
          const int j = jb + grp;
          const double dot = partial_dot(j, j < j1);
          if (j < j1) update(j, dot);
        }
    }
  };
  for (int c = 0; c < n; ++c) {
    const int par = c & 1;
    double* yc = Y + c * ld;
    const bool own_row = c >= r0 && c < r1;
    const int lo = max(c + 1 - r0, 0);
    if constexpr (PIV) {  // bring the largest remaining column (rows >= c) to position c
      const int lv = max(c - r0, 0);
      for (int jb = c; jb < nc; jb += QR_NG) {
        const int j = jb + grp;
        double s0 = 0.0;
        if (j < nc) {
          const double* yj = Y + j * ld;
          for (int i = lv + gl; i < nr; i += QR_GL) s0 = fma(yj[i], yj[i], s0);
        }
#pragma unroll
        for (int o = QR_GL / 2; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        if (j < nc && gl == 0) sh.nrm[j] = s0;
      }
      __syncthreads();
      if constexpr (CL) {
        csync();
        for (int j = c + tid; j < nc; j += QR_THREADS) {
          double t = 0.0;
          for (int r = 0; r < C; ++r) t += remote(&sh.nrm[j], r);
          sh.wsum[j] = t;
        }
        csync();
        for (int j = c + tid; j < nc; j += QR_THREADS) sh.nrm[j] = sh.wsum[j];
        __syncthreads();
      }
      if (warp == 0) {
        double best = -1.0;
        int bj = c;
        for (int j = c + lane; j < nc; j += 32) {
          const double v = sh.nrm[j];
          if (v > best) {
            best = v;
            bj = j;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (ob > best || (ob == best && oj < bj)) {
            best = ob;
            bj = oj;
          }
        }
        if (lane == 0) sh.jmax = bj;
      }
      __syncthreads();
      const int jm = sh.jmax;
      if (jm != c) {
        double* yj = Y + jm * ld;
        for (int i = tid; i < nr; i += QR_THREADS) {
          const double t = yc[i];
          yc[i] = yj[i];
          yj[i] = t;
        }
      }
      __syncthreads();
    }
    // reflector of column c (warp 0)
    if (warp == 0) {
      double ss = 0.0;
      for (int i = lo + lane; i < nr; i += 32) ss = fma(yc[i], yc[i], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) {
        sh.a[par][0] = ss;
        sh.a[par][1] = own_row ? yc[c - r0] : 0.0;
      }
    }
    csync();
    if (warp == 0) {
      // lanes q < C load rank q's partial (in flight together), summed in rank order
      double part = lane < C ? remote(&sh.a[par][0], lane) : 0.0;
      double sst = 0.0;
      for (int q = 0; q < C; ++q) sst += __shfl_sync(0xffffffffu, part, q);
      double alpha = lane == 0 ? remote(&sh.a[par][1], c / R) : 0.0;
      alpha = __shfl_sync(0xffffffffu, alpha, 0);
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
      for (int i = lo + lane; i < nr; i += 32) yc[i] *= scal;
      if (lane == 0) {
        if (own_row) yc[c - r0] = beta;
        sh.tau[c] = tc;
        sh.rdiag[c] = beta;
      }
    }
    __syncthreads();
    apply_reflector(c, c + 1, nc, par);
    __syncthreads();
  }
  // range-finder check: |(I - Q Q^T) y_probe|^2 = sum of the probe columns' rows >= n
  double pres = 0.0;
  {
    const int lo = max(n - r0, 0);
    if (warp < d.p) {
      const double* yq = Y + (n + warp) * ld;
      double ss = 0.0;
      for (int i = lo + lane; i < nr; i += 32) ss = fma(yq[i], yq[i], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) sh.w[0][QR_MAXN + warp] = ss;
    }
    __syncthreads();
    csync();
    for (int q = 0; q < d.p; ++q) {
      double t = 0.0;
      for (int r = 0; r < C; ++r) t += remote(&sh.w[0][QR_MAXN + q], r);
      pres = fmax(pres, sqrt(t));
    }
    csync();
  }
  // Q in place (dorg2r): backward over the reflectors; column c + 1 becomes Q's column
  // (its reflector no longer read) at the start of step c
  auto finish_col = [&](int c) {
    double* y = Y + c * ld;
    const double tc = sh.tau[c];
    for (int i = tid; i < nr; i += QR_THREADS) {
      const int gi = r0 + i;
      y[i] = gi < c ? 0.0 : (gi == c ? 1.0 - tc : -tc * y[i]);
    }
  };
  for (int c = n - 1; c >= 0; --c) {
    if (c + 1 < n) {
      finish_col(c + 1);
      __syncthreads();
    }
    apply_reflector(c, c + 1, n, c & 1);
    __syncthreads();
  }
  finish_col(0);
  __syncthreads();
  for (int jj = 0; jj < n; ++jj)
    for (int i = tid; i < nr; i += QR_THREADS) d.Q[r0 + i + (long long)jj * d.ldq] = Y[i + jj * ld];
  if (rank == 0 && d.stat) {
    double dmax = 0.0;
    if (d.S)
      for (int i = tid; i < d.nbs; i += QR_THREADS) dmax = fmax(dmax, fabs(d.S[i + (long long)i * d.lds]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) sh.red[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_WARPS; ++w) t = fmax(t, sh.red[w]);
      const double eps = *eps_ptr;
      // operator scale (sketch factors) or, without S, the leading |R_00| (rank-revealing QR)
      const double scale = d.S ? t * sqrt(double(d.k) / 3.0) : (n > 0 ? fabs(sh.rdiag[0]) : 0.0);
      int rk = 0;
      for (int i = 0; i < n; ++i)
        if (fabs(sh.rdiag[i]) > eps * scale) ++rk;
      d.stat[0] = double(rk);
      d.stat[1] = scale > 0.0 ? pres / scale : 0.0;
    }
  }
  csync();  // no CTA leaves while others may still read its shared memory
}

// The sketch factors' Householder QR with ONE cluster reduction per column step
// (hqr_kernel above needs two, plus one per step of the Q formation): step c
// reduces, for every trailing column j >= c, s_j = sum_{i > c} y_ic y_ij
// (s_c = |x(c+1:)|^2) together with row c's entries y_cj; every CTA then forms
// beta, tau and v = [1; y(c+1:, c) / (alpha - beta)] itself from the same sums in
// rank order (bit-identical reflectors on every CTA) and
// v^T y_j = y_cj + s_j / (alpha - beta). The reflector column is scaled lazily
// at the next step (no CTA reads it there). The explicit Q is formed backward
// (dorg2r) with the same one-reduction step; the C partials of a sum are loaded
// together (DSMEM loads in flight at once) and added in rank order.
template <bool CL, bool SM>
__global__ void __launch_bounds__(QR_THREADS) hqr1_kernel(const QrDesc* __restrict__ descs,
                                                          const double* eps_ptr, int C) {
  extern __shared__ __align__(16) double qdyn[];
  __shared__ double part[2][QR_MAXN + 8];        // [parity] this CTA's partial sums (+ probe norms)
  __shared__ double rowc[2][QR_MAXN];            // [parity] row c of the trailing columns (row owner)
  __shared__ double tot[QR_MAXN], rct[QR_MAXN];  // cluster sums / row c, local copies
  __shared__ double tau_s[QR_MAXN], rdiag[QR_MAXN];
  __shared__ double red[QR_WARPS];
  const int rank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const QrDesc d = descs[blockIdx.x / C];
  const int m = d.m, n = d.n, nc = d.n + d.p;
  const int R = (m + C - 1) / C, r0 = rank * R, r1 = min(m, r0 + R), nr = max(r1 - r0, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gl = tid & (QR_GL - 1), grp = tid / QR_GL;
  const long long ld = SM ? (nr | 1) : d.ldy;
  double* Y = SM ? qdyn : d.Y + r0;  // local rows, column-major
  if constexpr (SM) {
    for (int j = 0; j < nc; ++j)
      for (int i = tid; i < nr; i += QR_THREADS) Y[i + j * ld] = d.Y[r0 + i + (long long)j * d.ldy];
    __syncthreads();
  }
  auto csync = [] {
    if constexpr (CL) cg::this_cluster().sync();
    else __syncthreads();
  };
  auto csum = [&](const double* slot) -> double {
    if constexpr (CL) {
      double v[QR_MAXC];
#pragma unroll
      for (int q = 0; q < QR_MAXC; ++q)
        v[q] = q < C ? *cg::this_cluster().map_shared_rank(const_cast<double*>(slot), q) : 0.0;
      double t = v[0];
#pragma unroll
      for (int q = 1; q < QR_MAXC; ++q)
        if (q < C) t += v[q];
      return t;
    } else {
      return *slot;
    }
  };
  // partial dot of local rows [lo, nr) of columns a and b by the 8 lanes of a group
  auto gdot = [&](const double* ya, const double* yb, int lo, bool valid) {
    double s0 = 0.0, s1 = 0.0;
    if (valid) {
      int i = lo + gl;
      for (; i + QR_GL < nr; i += 2 * QR_GL) {
        s0 = fma(ya[i], yb[i], s0);
        s1 = fma(ya[i + QR_GL], yb[i + QR_GL], s1);
      }
      if (i < nr) s0 = fma(ya[i], yb[i], s0);
    }
    double dot = s0 + s1;
#pragma unroll
    for (int o = QR_GL / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    return dot;
  };
  double scal_prev = 0.0, beta_prev = 0.0;
  auto finish_reflector = [&](int c) {  // column c <- [beta; v(c+1:)]
    const int lo = max(c + 1 - r0, 0);
    double* y = Y + c * ld;
    for (int i = lo + tid; i < nr; i += QR_THREADS) y[i] *= scal_prev;
    if (tid == 0 && c >= r0 && c < r1) y[c - r0] = beta_prev;
  };
  for (int c = 0; c < n; ++c) {
    const int par = c & 1;
    const int lo = max(c + 1 - r0, 0);
    const bool own = c >= r0 && c < r1;
    const double* yc = Y + c * ld;
    if (c > 0) finish_reflector(c - 1);
    for (int jb = c; jb < nc; jb += QR_NG) {
      const int j = jb + grp;
      const double dot = gdot(yc, Y + min(j, nc - 1) * ld, lo, j < nc);
      if (j < nc && gl == 0) part[par][j] = dot;
    }
    if (own)
      for (int j = c + tid; j < nc; j += QR_THREADS) rowc[par][j] = Y[(c - r0) + j * ld];
    csync();
    for (int j = c + tid; j < nc; j += QR_THREADS) {
      tot[j] = csum(&part[par][j]);
      if constexpr (CL) rct[j] = *cg::this_cluster().map_shared_rank(&rowc[par][j], c / R);
      else rct[j] = rowc[par][j];
    }
    __syncthreads();
    const double sst = tot[c], alpha = rct[c];
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
    if (tid == 0) {
      tau_s[c] = tc;
      rdiag[c] = beta;
    }
    if (tc != 0.0)
      for (int jb = c + 1; jb < nc; jb += QR_NG) {
        const int j = jb + grp;
        if (j < nc) {
          const double f = tc * fma(scal, tot[j], rct[j]);  // tau v^T y_j
          const double g = f * scal;
          double* yj = Y + j * ld;
          if (own && gl == 0) yj[c - r0] -= f;
          for (int i = lo + gl; i < nr; i += QR_GL) yj[i] = fma(-g, yc[i], yj[i]);
        }
      }
    scal_prev = scal;
    beta_prev = beta;
    __syncthreads();
  }
  if (n > 0) finish_reflector(n - 1);
  __syncthreads();
  // range-finder check: |(I - Q Q^T) y_probe|^2 = sum of the probe columns' rows >= n
  double pres = 0.0;
  {
    const int lo = max(n - r0, 0);
    if (warp < d.p) {
      const double* yq = Y + (n + warp) * ld;
      double ss = 0.0;
      for (int i = lo + lane; i < nr; i += 32) ss = fma(yq[i], yq[i], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) part[0][QR_MAXN + warp] = ss;
    }
    csync();
    for (int q = 0; q < d.p; ++q) pres = fmax(pres, sqrt(csum(&part[0][QR_MAXN + q])));
    csync();  // the probe slots are free again
  }
  // Q in place (dorg2r): backward over the reflectors. Before H_c is applied, the
  // columns j > c are zero in rows <= c, so v^T q_j = sum_{i > c} v_i q_ij.
  auto finish_col = [&](int c) {
    double* y = Y + c * ld;
    const double tc = tau_s[c];
    for (int i = tid; i < nr; i += QR_THREADS) {
      const int gi = r0 + i;
      y[i] = gi < c ? 0.0 : (gi == c ? 1.0 - tc : -tc * y[i]);
    }
  };
  for (int c = n - 1; c >= 0; --c) {
    const int par = c & 1;
    const int lo = max(c + 1 - r0, 0);
    const bool own = c >= r0 && c < r1;
    const double* yc = Y + c * ld;
    const double tc = tau_s[c];
    if (c + 1 < n) {
      finish_col(c + 1);
      __syncthreads();
    }
    for (int jb = c + 1; jb < n; jb += QR_NG) {
      const int j = jb + grp;
      const double dot = gdot(yc, Y + min(j, n - 1) * ld, lo, j < n);
      if (j < n && gl == 0) part[par][j] = dot;
    }
    csync();
    for (int j = c + 1 + tid; j < n; j += QR_THREADS) tot[j] = csum(&part[par][j]);
    __syncthreads();
    if (tc != 0.0)
      for (int jb = c + 1; jb < n; jb += QR_NG) {
        const int j = jb + grp;
        if (j < n) {
          const double f = tc * tot[j];
          double* yj = Y + j * ld;
          if (own && gl == 0) yj[c - r0] = -f;
          for (int i = lo + gl; i < nr; i += QR_GL) yj[i] = fma(-f, yc[i], yj[i]);
        }
      }
    __syncthreads();
  }
  if (n > 0) finish_col(0);
  __syncthreads();
  for (int jj = 0; jj < n; ++jj)
    for (int i = tid; i < nr; i += QR_THREADS) d.Q[r0 + i + (long long)jj * d.ldq] = Y[i + jj * ld];
  if (rank == 0 && d.stat) {
    double dmax = 0.0;
    if (d.S)
      for (int i = tid; i < d.nbs; i += QR_THREADS) dmax = fmax(dmax, fabs(d.S[i + (long long)i * d.lds]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) red[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_WARPS; ++w) t = fmax(t, red[w]);
      const double eps = *eps_ptr;
      const double scale = d.S ? t * sqrt(double(d.k) / 3.0) : (n > 0 ? fabs(rdiag[0]) : 0.0);
      int rk = 0;
      for (int i = 0; i < n; ++i)
        if (fabs(rdiag[i]) > eps * scale) ++rk;
      d.stat[0] = double(rk);
      d.stat[1] = scale > 0.0 ? pres / scale : 0.0;
    }
  }
  if constexpr (CL) cg::this_cluster().sync();  // no CTA leaves while others may still read its shared memory
}

// ---------------------------------------------------------------------------
// hqrb_kernel: the sketch factors' Householder QR BLOCKED (dgeqrf / dorgqr with
// compact-WY block reflectors, panels of QB = 16 columns). hqr_kernel / hqr1_kernel
// apply every reflector to every trailing column at once (level-2: each column step
// streams the whole trailing block through shared memory -- the measured bound);
// here a column step touches only its panel, and the trailing columns take one
// rank-16 update per panel: W = V^T Y (partials per CTA, summed over the cluster),
// Y -= V (T^T W) (dlarft's T). The explicit Q is formed backward per panel as
// Q[:, c0:] = [E | Q[:, c1:]] - V T (V^T [E | Q[:, c1:]]), E the panel's unit
// columns. Cluster sums are a reduce-scatter + all-gather through DSMEM (each CTA
// sums its 1/C share of the entries, then reads the others' shares), added in rank
// order so every CTA holds bit-identical sums. Results equal dgeqrf/dorgqr's up to
// rounding (same reflectors, beta = -sign(alpha) |x|, tau = (beta - alpha) / beta).
constexpr int QB = 16;
#ifdef HQRB_PROFILE
__device__ long long g_hqrb_clk[16];
__device__ unsigned long long g_hqrb_t[2 * 2048];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HCLK_T(v) long long v = clock64()
#define HCLK_ADD(slot, t0) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_hqrb_clk[slot] += clock64() - (t0); } while (0)
#else
#define HCLK_T(v) do { } while (0)
#define HCLK_ADD(slot, t0) do { } while (0)
#endif

struct HqrbSmem {  // dynamic shared-memory carve (doubles), identical for every CTA of a launch
  int ldl, rmax, ncmax, npan, wcols;
  __host__ __device__ long long y() const { return 0; }
  __host__ __device__ long long vr() const { return (long long)ldl * ncmax; }
  __host__ __device__ long long wp() const { return vr() + (long long)rmax * QB; }
  __host__ __device__ long long ws() const { return wp(); }  // the sums overwrite the partials (see allreduce_w)
  __host__ __device__ long long ts() const { return wp() + (long long)QB * wcols; }
  __host__ __device__ long long total() const { return ts() + (long long)npan * QB * QB; }
};

template <bool CL>
__global__ void __launch_bounds__(QR_THREADS) hqrb_kernel(const QrDesc* __restrict__ descs, const double* eps_ptr,
                                                          int C, HqrbSmem L) {
#ifdef HQRB_PROFILE
  if (threadIdx.x == 0) g_hqrb_t[2 * blockIdx.x] = gtimer();
#endif
  extern __shared__ __align__(16) double qdyn[];
  __shared__ double part[2][QB + 8];  // [parity] column-step partials (+ probe norms)
  __shared__ double rowc[2][QB];
  __shared__ double tot[QB], rct[QB];
  __shared__ double tau_s[QR_MAXN], rdiag[QR_MAXN];
  __shared__ double red[QR_WARPS];
  const int rank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const QrDesc d = descs[blockIdx.x / C];
  const int m = d.m, n = d.n, nc = d.n + d.p;
  const int R = (m + C - 1) / C, r0 = rank * R, r1 = min(m, r0 + R), nr = max(r1 - r0, 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = L.ldl;
  double* Y = qdyn + L.y();
  double* Vr = qdyn + L.vr();  // [rmax][QB] row-major: the panel's reflectors, local rows
  double* Wp = qdyn + L.wp();  // [QB][wcols] this CTA's partial sums
  double* Ws = qdyn + L.ws();  // [QB][wcols] cluster sums
  double* Ts = qdyn + L.ts();  // [npan][QB][QB] T of every panel (upper triangular)
  for (int j = 0; j < nc; ++j)
    for (int i = tid; i < nr; i += QR_THREADS) Y[i + j * ld] = d.Y[r0 + i + (long long)j * d.ldy];
  __syncthreads();
  auto csync = [] {
    if constexpr (CL) cg::this_cluster().sync();
    else __syncthreads();
  };
  auto r0_glob = [&](int r) { return r0 + r; };  // local row -> global row
  auto rsum = [&](const double* slot) -> double {  // sum over the cluster's copies of *slot, rank order
    if constexpr (CL) {
      double v[QR_MAXC];
#pragma unroll
      for (int q = 0; q < QR_MAXC; ++q)
        v[q] = q < C ? *cg::this_cluster().map_shared_rank(const_cast<double*>(slot), q) : 0.0;
      double t = v[0];
#pragma unroll
      for (int q = 1; q < QR_MAXC; ++q)
        if (q < C) t += v[q];
      return t;
    } else {
      return *slot;
    }
  };
  // Ws[0 : QB * cols) = cluster sum of Wp, in place (Ws aliases Wp): reduce-scatter (CTA q
  // sums share q over every CTA's partials and stores it in its own share-q slots, which no
  // other CTA reads in this phase), barrier, all-gather (CTA q copies every other share
  // from its owner into its own slots, which no other CTA reads in this phase)
  auto allreduce_w = [&](int cols) {
    const int cnt = QB * cols;
    csync();  // every partial written
    if constexpr (CL) {
      const int share = (cnt + C - 1) / C, e0 = rank * share, e1 = min(cnt, e0 + share);
      for (int e = e0 + tid; e < e1; e += QR_THREADS) {
        const int k = (e % QB) * L.wcols + e / QB;
        Ws[k] = rsum(&Wp[k]);  // element k of share `rank`: read (everywhere) and written (here) by this thread only
      }
      cg::this_cluster().sync();
      for (int q = 0; q < C; ++q) {
        if (q == rank) continue;
        const int f0 = q * share, f1 = min(cnt, f0 + share);
        const double* rws = cg::this_cluster().map_shared_rank(Ws, q);
        for (int e = f0 + tid; e < f1; e += QR_THREADS) {
          const int k = (e % QB) * L.wcols + e / QB;
          Ws[k] = rws[k];
        }
      }
      // every CTA has copied every share before anybody overwrites its own (the caller
      // transforms the sums in place)
      cg::this_cluster().sync();
    } else {
      for (int e = tid; e < cnt; e += QR_THREADS) Ws[(e % QB) * L.wcols + e / QB] = Wp[(e % QB) * L.wcols + e / QB];
    }
    __syncthreads();
  };
  // Vr <- the local rows of panel [c0, c1)'s reflectors (unit diagonal, zeros above)
  auto stage_v = [&](int c0, int c1) {
    for (int e = tid; e < nr * QB; e += QR_THREADS) {
      const int i = e / QB, cc = e % QB, c = c0 + cc, gi = r0 + i;
      Vr[i * QB + cc] = (c >= c1 || gi < c) ? 0.0 : (gi == c ? 1.0 : Y[i + c * ld]);
    }
    __syncthreads();
  };
  // ---- the panel products on the FP64 tensor pipe (mma.sync.m16n8k4), warps over 8-column
  // tiles. W[:, wofs + t] = V^T x_t over the local rows, x_t = column t of Vr (vcols) or of
  // Y at ycols (ld)
  const int g8 = lane >> 2, t4 = lane & 3;
  auto mma_w = [&](const double* ycols, bool vcols, int ncols, int wofs) {
    const int ntile = (ncols + 7) / 8;
    for (int tile = warp; tile < ntile; tile += QR_WARPS) {
      const int cb = tile * 8, col = cb + g8;
      const bool cv = col < ncols;
      const double* yc = ycols + (long long)min(col, max(ncols - 1, 0)) * ld;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k0 = 0; k0 < nr; k0 += 4) {
        const int r = k0 + t4;
        const bool rv = r < nr;
        const double a0 = rv ? Vr[r * QB + g8] : 0.0;
        const double a1 = rv ? Vr[r * QB + g8 + 8] : 0.0;
        const double b0 = (rv && cv) ? (vcols ? Vr[r * QB + col] : yc[r]) : 0.0;
        mma_f64_m16n8k4(acc, a0, a1, b0);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int cc = g8 + 8 * (v >> 1), cl = cb + 2 * t4 + (v & 1);
        if (cl < ncols) Wp[cc * L.wcols + wofs + cl] = acc[v];
      }
    }
  };
  // out[:, t] = base_t - V Ws[:, wofs + t] over the local rows, base_t = column t of Y at
  // ycols (in place) or, unit, the unit vector of global row c_unit + t
  auto mma_upd = [&](double* ycols, int ncols, int wofs, bool unit, int c_unit) {
    const int rt = (nr + 15) / 16, ct = (ncols + 7) / 8;
    for (int tile = warp; tile < rt * ct; tile += QR_WARPS) {
      const int r0 = (tile % rt) * 16, cb = (tile / rt) * 8;
      double acc[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = r0 + g8 + 8 * (v >> 1), cl = cb + 2 * t4 + (v & 1);
        acc[v] = (r < nr && cl < ncols) ? (unit ? (r0_glob(r) == c_unit + cl ? 1.0 : 0.0) : ycols[r + (long long)cl * ld])
                                        : 0.0;
      }
      const int cl = cb + g8;
#pragma unroll
      for (int k0 = 0; k0 < QB; k0 += 4) {
        const double a0 = (r0 + g8 < nr) ? -Vr[(r0 + g8) * QB + k0 + t4] : 0.0;
        const double a1 = (r0 + g8 + 8 < nr) ? -Vr[(r0 + g8 + 8) * QB + k0 + t4] : 0.0;
        const double b0 = cl < ncols ? Ws[(k0 + t4) * L.wcols + wofs + cl] : 0.0;
        mma_f64_m16n8k4(acc, a0, a1, b0);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = r0 + g8 + 8 * (v >> 1), c2 = cb + 2 * t4 + (v & 1);
        if (r < nr && c2 < ncols) ycols[r + (long long)c2 * ld] = acc[v];
      }
    }
  };
  const int gl = tid & 15, grp = tid >> 4;  // 16 groups of 16 lanes: one panel column per group
  const int npan = (n + QB - 1) / QB;
  for (int pn = 0; pn < npan; ++pn) {
    const int c0 = pn * QB, c1 = min(n, c0 + QB), bw = c1 - c0;
    double scal_prev = 0.0, beta_prev = 0.0;
    HCLK_T(tp0);
    for (int c = c0; c < c1; ++c) {
      const int par = c & 1;
      const int lo = max(c + 1 - r0, 0);
      const bool own = c >= r0 && c < r1;
      const double* yc = Y + c * ld;
      if (c > c0) {  // the previous reflector column: [beta; v]
        const int lp = max(c - r0, 0);
        double* yp = Y + (c - 1) * ld;
        for (int i = lp + tid; i < nr; i += QR_THREADS) yp[i] *= scal_prev;
        if (tid == 0 && c - 1 >= r0 && c - 1 < r1) yp[c - 1 - r0] = beta_prev;
      }
      {
        const int j = c + grp;
        double s0 = 0.0;
        if (j < c1) {
          const double* yj = Y + j * ld;
          for (int i = lo + gl; i < nr; i += 16) s0 = fma(yc[i], yj[i], s0);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        if (j < c1 && gl == 0) part[par][grp] = s0;
        if (own && tid < c1 - c) rowc[par][tid] = Y[(c - r0) + (c + tid) * ld];
      }
      csync();
      if (tid < c1 - c) {
        tot[tid] = rsum(&part[par][tid]);
        if constexpr (CL) rct[tid] = *cg::this_cluster().map_shared_rank(&rowc[par][tid], c / R);
        else rct[tid] = rowc[par][tid];
      }
      __syncthreads();
      const double sst = tot[0], alpha = rct[0];
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
      if (tid == 0) {
        tau_s[c] = tc;
        rdiag[c] = beta;
      }
      if (tc != 0.0 && grp >= 1 && c + grp < c1) {
        const int j = c + grp;
        const double f = tc * fma(scal, tot[grp], rct[grp]);
        const double g = f * scal;
        double* yj = Y + j * ld;
        if (own && gl == 0) yj[c - r0] -= f;
        for (int i = lo + gl; i < nr; i += 16) yj[i] = fma(-g, yc[i], yj[i]);
      }
      scal_prev = scal;
      beta_prev = beta;
      __syncthreads();
    }
    {  // the panel's last reflector column
      const int c = c1 - 1, lp = max(c + 1 - r0, 0);
      double* yp = Y + c * ld;
      for (int i = lp + tid; i < nr; i += QR_THREADS) yp[i] *= scal_prev;
      if (tid == 0 && c >= r0 && c < r1) yp[c - r0] = beta_prev;
    }
    __syncthreads();
    // block reflector: G = V^T V and W = V^T Y[:, c1:nc] (one reduction), T (dlarft),
    // Y[:, c1:nc] -= V (T^T W)
    HCLK_ADD(1, tp0);
    HCLK_T(tp1);
    stage_v(c0, c1);
    const int nt = nc - c1, ncol = QB + nt;
    mma_w(nullptr, true, QB, 0);         // G = V^T V
    mma_w(Y + c1 * ld, false, nt, QB);   // W = V^T Y[:, c1:nc]
    allreduce_w(ncol);
    HCLK_ADD(2, tp1);
    HCLK_T(tp2);
    double* T = Ts + pn * QB * QB;  // T[i * QB + k]
    if (warp == 0 && lane < QB) {  // dlarft (forward, columnwise): T[0:k, k] = -tau_k T[0:k, 0:k] G[0:k, k]
      const int i = lane;             // lane i builds row i of T in registers
      double tr[QB];
#pragma unroll
      for (int k = 0; k < QB; ++k) {
        double g[QB];
#pragma unroll
        for (int l = 0; l < k; ++l) g[l] = Ws[l * L.wcols + k];  // G[0:k, k] (broadcast loads)
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int l = 0; l < k; ++l) {
          const double a = l >= i ? tr[l] : 0.0;
          if (l & 1) s1 = fma(a, g[l], s1);
          else s0 = fma(a, g[l], s0);
        }
        const double tk = k < bw ? tau_s[c0 + k] : 0.0;
        tr[k] = i < k ? -tk * (s0 + s1) : (i == k ? tk : 0.0);
      }
#pragma unroll
      for (int k = 0; k < QB; ++k) T[i * QB + k] = tr[k];
    }
    __syncthreads();
    HCLK_ADD(3, tp2);
    HCLK_T(tp3);
    for (int t = tid; t < nt; t += QR_THREADS) {  // W <- T^T W in place, column by column
      double w[QB];
#pragma unroll
      for (int cc = 0; cc < QB; ++cc) w[cc] = Ws[cc * L.wcols + QB + t];
#pragma unroll
      for (int cc = 0; cc < QB; ++cc) {
        double sacc = 0.0;
#pragma unroll
        for (int l = 0; l <= cc; ++l) sacc = fma(T[l * QB + cc], w[l], sacc);
        Ws[cc * L.wcols + QB + t] = sacc;
      }
    }
    __syncthreads();
    mma_upd(Y + c1 * ld, nt, QB, false, 0);
    __syncthreads();
    HCLK_ADD(4, tp3);
  }
  HCLK_T(tp4);
  // range-finder check: |(I - Q Q^T) y_probe|^2 = sum of the probe columns' rows >= n
  double pres = 0.0;
  {
    const int lo = max(n - r0, 0);
    if (warp < d.p) {
      const double* yq = Y + (n + warp) * ld;
      double ss = 0.0;
      for (int i = lo + lane; i < nr; i += 32) ss = fma(yq[i], yq[i], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) part[0][QB + warp] = ss;
    }
    csync();
    for (int q = 0; q < d.p; ++q) pres = fmax(pres, sqrt(rsum(&part[0][QB + q])));
  }
  HCLK_ADD(5, tp4);
  HCLK_T(tp5);
  // Q, backward over the panels: Q[:, c0:n] = [E | Q[:, c1:n]] - V T (V^T [E | Q[:, c1:n]])
  for (int pn = npan - 1; pn >= 0; --pn) {
    const int c0 = pn * QB, c1 = min(n, c0 + QB);
    stage_v(c0, c1);
    const int nq = n - c1, ncol = QB + nq;
    if (tid < QB) {  // V^T E = V1^T: the owner's rows c0 + tid
      const int gi = c0 + tid;
      const bool mine = gi >= r0 && gi < r1 && gi < c1;
#pragma unroll
      for (int cc = 0; cc < QB; ++cc) Wp[cc * L.wcols + tid] = mine ? Vr[(gi - r0) * QB + cc] : 0.0;
    }
    mma_w(Y + c1 * ld, false, nq, QB);  // V^T Q[:, c1:n]
    allreduce_w(ncol);
    const double* T = Ts + pn * QB * QB;
    for (int t = tid; t < ncol; t += QR_THREADS) {  // W <- T W in place (T upper)
      double w[QB];
#pragma unroll
      for (int cc = 0; cc < QB; ++cc) w[cc] = Ws[cc * L.wcols + t];
#pragma unroll
      for (int cc = 0; cc < QB; ++cc) {
        double sacc = 0.0;
#pragma unroll
        for (int l = cc; l < QB; ++l) sacc = fma(T[cc * QB + l], w[l], sacc);
        Ws[cc * L.wcols + t] = sacc;
      }
    }
    __syncthreads();
    mma_upd(Y + c1 * ld, nq, QB, false, 0);               // formed columns, in place
    mma_upd(Y + c0 * ld, c1 - c0, 0, true, c0);           // the panel's own columns from E
    __syncthreads();
  }
  HCLK_ADD(6, tp5);
  for (int jj = 0; jj < n; ++jj)
    for (int i = tid; i < nr; i += QR_THREADS) d.Q[r0 + i + (long long)jj * d.ldq] = Y[i + jj * ld];
  if (rank == 0 && d.stat) {
    double dmax = 0.0;
    if (d.S)
      for (int i = tid; i < d.nbs; i += QR_THREADS) dmax = fmax(dmax, fabs(d.S[i + (long long)i * d.lds]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) red[warp] = dmax;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < QR_WARPS; ++w) t = fmax(t, red[w]);
      const double eps = *eps_ptr;
      const double scale = d.S ? t * sqrt(double(d.k) / 3.0) : (n > 0 ? fabs(rdiag[0]) : 0.0);
      int rk = 0;
      for (int i = 0; i < n; ++i)
        if (fabs(rdiag[i]) > eps * scale) ++rk;
      d.stat[0] = double(rk);
      d.stat[1] = scale > 0.0 ? pres / scale : 0.0;
    }
  }
#ifdef HQRB_PROFILE
  if (threadIdx.x == 0) g_hqrb_t[2 * blockIdx.x + 1] = gtimer();
#endif
  if constexpr (CL) cg::this_cluster().sync();  // no CTA leaves while others may still read its shared memory
}

// ---------------------------------------------------------------------------
constexpr int HP_THREADS = 1024, HP_WARPS = HP_THREADS / 32, HP_NG = HP_THREADS / QR_GL;
// hqrp_kernel: the rank-revealing Householder QR with column pivoting of the HBS
// compression (hqr_kernel<., ., PIV>'s reflectors, pivot rule and rank count), one
// CTA per matrix in shared memory. Per column step: one block argmax over the
// maintained trailing-column norms, the swap, the reflector (every warp forms it
// from the same column, no barrier), then groups of 8 lanes own the trailing
// columns: dot product, update and the EXACT new norm of rows > c in one pass (the
// values are in registers while written: no norm recomputation sweep, no
// downdating). Q is formed in place (dorg2r).
__global__ void __launch_bounds__(HP_THREADS) hqrp_kernel(const QrDesc* __restrict__ descs, const double* eps_ptr) {
  extern __shared__ __align__(16) double qdyn[];
  __shared__ double nrm[QR_MAXN];
  __shared__ double tau_s[QR_MAXN], rdiag[QR_MAXN];
  __shared__ double wbest[HP_WARPS];
  __shared__ int wj[HP_WARPS];
  __shared__ int rank_s;
  HCLK_T(tq0);
  const QrDesc d = descs[blockIdx.x];
  const int m = d.m, n = d.n, nc = d.n + d.p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gl = tid & (QR_GL - 1), grp = tid / QR_GL;  // HP_NG groups of 8 lanes
  const int ld = m | 1;
  double* Y = qdyn;
  for (int e = tid; e < m * nc; e += HP_THREADS) {  // every thread: one latency round, not one per column
    const int i = e % m, j = e / m;
    Y[i + j * ld] = d.Y[i + (long long)j * d.ldy];
  }
  __syncthreads();
  // initial column norms (rows >= 0)
  for (int jb = 0; jb < nc; jb += HP_NG) {
    const int j = jb + grp;
    double s0 = 0.0;
    if (j < nc)
      for (int i = gl; i < m; i += QR_GL) s0 = fma(Y[i + j * ld], Y[i + j * ld], s0);
#pragma unroll
    for (int o = QR_GL / 2; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    if (j < nc && gl == 0) nrm[j] = s0;
  }
  __syncthreads();
  HCLK_ADD(7, tq0);
  double scal_prev = 0.0, beta_prev = 0.0;
  for (int c = 0; c < n; ++c) {
    HCLK_T(tqa);
    // (a) pivot: the largest remaining norm, lowest index on ties
    {
      double best = -1.0;
      int bj = 0x7fffffff;
      for (int j = c + tid; j < nc; j += HP_THREADS) {
        const double v = nrm[j];
        if (v > best) {
          best = v;
          bj = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob > best || (ob == best && oj < bj)) {
          best = ob;
          bj = oj;
        }
      }
      if (lane == 0) {
        wbest[warp] = best;
        wj[warp] = bj;
      }
      // the previous reflector column: [beta; v] (no CTA reads it in this step)
      if (c > 0) {
        double* yp = Y + (c - 1) * ld;
        for (int i = c + tid; i < m; i += HP_THREADS) yp[i] *= scal_prev;
        if (tid == 0 && c - 1 < m) yp[c - 1] = beta_prev;
      }
    }
    __syncthreads();
    int jm;
    {  // every warp reduces the per-warp winners with shuffles (no serial loop over warps)
      double b = lane < HP_WARPS ? wbest[lane] : -1.0;
      int bj = lane < HP_WARPS ? wj[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob > b || (ob == b && oj < bj)) {
          b = ob;
          bj = oj;
        }
      }
      jm = bj;
    }
    HCLK_ADD(8, tqa);
    HCLK_T(tqb);
    // (b) swap columns c <-> jm
    if (jm != c) {
      double* yc = Y + c * ld;
      double* yj = Y + jm * ld;
      for (int i = tid; i < m; i += HP_THREADS) {
        const double t = yc[i];
        yc[i] = yj[i];
        yj[i] = t;
      }
    }
    __syncthreads();
    if (jm != c && tid == 0) {
      const double t = nrm[c];
      nrm[c] = nrm[jm];
      nrm[jm] = t;
    }
    HCLK_ADD(9, tqb);
    HCLK_T(tqc);
    // (c) the reflector of column c, formed by every warp (identical sums)
    const double* yc = Y + c * ld;
    double ss = 0.0;
    for (int i = c + 1 + lane; i < m; i += 32) ss = fma(yc[i], yc[i], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double alpha = c < m ? yc[c] : 0.0;
    double beta, tc, scal;
    if (ss == 0.0) {
      beta = alpha;
      tc = 0.0;
      scal = 0.0;
    } else {
      beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
      tc = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tid == 0) {
      tau_s[c] = tc;
      rdiag[c] = beta;
    }
    // (d) trailing columns: v^T y_j = y_cj + scal sum_{i > c} x_i y_ij; update; new norms
    for (int jb = c + 1; jb < nc; jb += HP_NG) {
      const int j = jb + grp;
      const bool live = j < nc;
      double* yj = Y + (live ? j : c) * ld;
      double s0 = 0.0;
      if (live)
        for (int i = c + 1 + gl; i < m; i += QR_GL) s0 = fma(yc[i], yj[i], s0);
#pragma unroll
      for (int o = QR_GL / 2; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      double n2 = 0.0;
      if (live) {
        const double f = tc * fma(scal, s0, yj[c]);
        const double g = f * scal;
        for (int i = c + 1 + gl; i < m; i += QR_GL) {
          const double y = fma(-g, yc[i], yj[i]);
          yj[i] = y;
          n2 = fma(y, y, n2);
        }
      }
#pragma unroll
      for (int o = QR_GL / 2; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      if (live && gl == 0) {
        yj[c] -= tc * fma(scal, s0, yj[c]);
        nrm[j] = n2;
      }
    }
    scal_prev = scal;
    beta_prev = beta;
    __syncthreads();
    HCLK_ADD(10, tqc);
  }
  HCLK_T(tqd);
  if (n > 0) {
    double* yp = Y + (n - 1) * ld;
    for (int i = n + tid; i < m; i += HP_THREADS) yp[i] *= scal_prev;
    if (tid == 0 && n - 1 < m) yp[n - 1] = beta_prev;
  }
  if (tid == 0) {
    const double eps = *eps_ptr;
    const double scale = n > 0 ? fabs(rdiag[0]) : 0.0;
    int rk = 0;
    for (int i = 0; i < n; ++i)
      if (fabs(rdiag[i]) > eps * scale) ++rk;
    rank_s = rk;
    if (d.stat) {
      d.stat[0] = double(rk);
      d.stat[1] = 0.0;
    }
  }
  __syncthreads();
  const int nq = n;  // every column: the caller keeps max(rank of the rows side, of the columns side)
  auto finish_col = [&](int c) {
    double* y = Y + c * ld;
    const double tc = tau_s[c];
    for (int i = tid; i < m; i += HP_THREADS) y[i] = i < c ? 0.0 : (i == c ? 1.0 - tc : -tc * y[i]);
  };
  for (int c = nq - 1; c >= 0; --c) {
    if (c + 1 < nq) {
      finish_col(c + 1);
      __syncthreads();
    }
    const double* yc = Y + c * ld;
    const double tc = tau_s[c];
    for (int jb = c + 1; jb < nq; jb += HP_NG) {
      const int j = jb + grp;
      const bool live = j < nq;
      double* yj = Y + (live ? j : c) * ld;
      double s0 = 0.0;
      if (live)
        for (int i = c + 1 + gl; i < m; i += QR_GL) s0 = fma(yc[i], yj[i], s0);
#pragma unroll
      for (int o = QR_GL / 2; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      if (live && tc != 0.0) {
        const double f = tc * s0;
        if (gl == 0) yj[c] = -f;
        for (int i = c + 1 + gl; i < m; i += QR_GL) yj[i] = fma(-f, yc[i], yj[i]);
      }
    }
    __syncthreads();
  }
  if (nq > 0) finish_col(0);
  __syncthreads();
  HCLK_ADD(11, tqd);
  for (int e = tid; e < m * nq; e += HP_THREADS) {
    const int i = e % m, jj = e / m;
    d.Q[i + (long long)jj * d.ldq] = Y[i + jj * ld];
  }
}

// launch geometry of hqrb_kernel: the smallest cluster whose row blocks and work
// buffers fit in shared memory, widened while the launch leaves SMs idle
template <bool CL>
__global__ void hqrb_kernel(const QrDesc* __restrict__, const double*, int, HqrbSmem);
constexpr int HQRB_SMEM_MIN = 120 * 1024;  // one CTA per SM (co-resident CTAs would share its issue slots)
constexpr int HQRB_SMEM_MAX = 220 * 1024;

// clusters of C CTAs (one per SM) that can be resident at once, per device
static int hqrb_max_clusters(int C) {
  static int cache[8][5];
  static bool init[8][5];
  int dev = 0;
  cudaGetDevice(&dev);
  int li = 0;
  while ((1 << li) < C) ++li;
  if (dev < 8 && li < 5 && init[dev][li]) return cache[dev][li];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(QR_THREADS);
  cfg.dynamicSmemBytes = HQRB_SMEM_MIN;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, C > 1 ? (void*)hqrb_kernel<true> : (void*)hqrb_kernel<false>, &cfg) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    n = 0;
  }
  if (dev < 8 && li < 5) {
    cache[dev][li] = n;
    init[dev][li] = true;
  }
  return n;
}

// launch geometry of hqrb_kernel: the widest cluster (<= 16 CTAs, >= 32 rows each) whose
// row blocks and work buffers fit in shared memory and whose clusters are all resident at
// once; else the narrowest that fits
static bool hqrb_shape(int count, int max_m, int max_nc, int* C_out, HqrbSmem* L) {
  auto layout = [&](int C) {
    HqrbSmem s;
    s.rmax = (max_m + C - 1) / C;
    s.ldl = s.rmax | 1;
    s.ncmax = max_nc;
    s.npan = (max_nc + QB - 1) / QB;
    s.wcols = max_nc + QB;
    return s;
  };
  int best = 0;
  for (int C = 1; C <= QR_MAXC; C *= 2) {
    if (layout(C).total() * 8 > HQRB_SMEM_MAX) continue;
    if (best == 0) best = C;  // the narrowest that fits
    if (C > 1 && (max_m + C - 1) / C < 32) break;
    if (count <= hqrb_max_clusters(C)) best = C;
  }
  if (best == 0) return false;
  *C_out = best;
  *L = layout(best);
  return true;
}

// the K-slices of the structured boxes' sketches summed into Y1 / Y2 (slice 0 is Y itself)
__global__ void __launch_bounds__(256) sum_partials_kernel(const SumDesc* __restrict__ descs) {
  const SumDesc d = descs[blockIdx.y];
  const int total = d.m * d.n;
  for (int e = blockIdx.x * 256 + threadIdx.x; e < total; e += gridDim.x * 256) {
    const int r = e % d.m, c = e / d.m;
    double t = d.dst[r + (long long)c * d.ldd];
    for (int q = 0; q < d.slices; ++q) t += d.src[q * d.stride + r + (long long)c * d.lds];
    d.dst[r + (long long)c * d.ldd] = t;
  }
}

cudaError_t launch_sum_partials(const SumDesc* d_descs, int count, long long max_elems, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid(unsigned(std::min<long long>((max_elems + 255) / 256, 64)), count);
  sum_partials_kernel<<<grid, 256, 0, st>>>(d_descs);
  return cudaGetLastError();
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

// cluster size for an m x nc matrix: the smallest C whose row blocks fit in shared
// memory, else 16 CTAs working on the matrix in place (global memory, L1/L2-resident)
static int qr_cluster(int m, int nc, bool* sm) {
  for (int C = 1; C <= QR_MAXC; C *= 2) {
    const long long R = (m + C - 1) / C;
    if ((R | 1) * nc * 8 <= 200 * 1024) {
      *sm = true;
      return C;
    }
  }
  *sm = false;
  return QR_MAXC;
}

// DTN_HQR_FUSED=1: the sketch QR by hqr1_kernel (one reduction per column step; measured
// no faster than hqr_kernel: both are bound by the shared-memory traffic of the
// unblocked column updates, not by the cluster barriers)
static bool hqr_legacy() {
  static const bool on = std::getenv("DTN_HQR_FUSED") == nullptr;
  return on;
}

// DTN_HQR_BLOCKED=0: the unblocked sketch QR (hqr_kernel, or hqr1_kernel with DTN_HQR_FUSED)
static bool hqrb_off() {
  static const bool off = [] {
    const char* e = std::getenv("DTN_HQR_BLOCKED");
    return e && std::atoi(e) == 0;
  }();
  return off;
}

// DTN_HQRP=0: the pivoted QR by hqr_kernel<., ., true>
static bool hqrp_off() {
  static const bool off = [] {
    const char* e = std::getenv("DTN_HQRP");
    return e && std::atoi(e) == 0;
  }();
  return off;
}

cudaError_t struct_init() {
  {
    cudaError_t e = cudaFuncSetAttribute(hqrp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {hqrb_kernel<true>, hqrb_kernel<false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, HQRB_SMEM_MAX);
    if (e != cudaSuccess) return e;
  }
  {
    cudaError_t e = cudaFuncSetAttribute(hqrb_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {hqr1_kernel<true, true>, hqr1_kernel<false, true>, hqr1_kernel<true, false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {hqr1_kernel<true, true>, hqr1_kernel<true, false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {hqr_kernel<true, true>, hqr_kernel<false, true>, hqr_kernel<true, false>,
                 hqr_kernel<true, true, true>, hqr_kernel<false, true, true>, hqr_kernel<true, false, true>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {hqr_kernel<true, true>, hqr_kernel<true, false>, hqr_kernel<true, true, true>,
                 hqr_kernel<true, false, true>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_hqr(const QrDesc* d_descs, int count, int max_m, int max_nc, const double* d_eps, cudaStream_t st,
                       bool pivoted) {
  if (count <= 0) return cudaSuccess;
  if (max_nc > QR_MAXN) return cudaErrorInvalidValue;
  bool sm = true;
  const int C = qr_cluster(max_m, max_nc, &sm);
  if (std::getenv("DTN_DEBUG_QR"))
    std::fprintf(stderr, "hqr: count %d max_m %d max_nc %d cluster %d smem %d pivoted %d\n", count, max_m, max_nc, C,
                 int(sm), int(pivoted));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * C);
  cfg.blockDim = dim3(QR_THREADS);
  cfg.stream = st;
  cfg.dynamicSmemBytes = sm ? size_t(((max_m + C - 1) / C) | 1) * max_nc * 8 : 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  if (pivoted) {
    if (C == 1 && sm && !hqrp_off()) {
      cfg.dynamicSmemBytes = size_t(max_m | 1) * max_nc * 8;
      cfg.blockDim = dim3(HP_THREADS);
      return cudaLaunchKernelEx(&cfg, hqrp_kernel, d_descs, d_eps);
    }
    if (!sm) return cudaLaunchKernelEx(&cfg, hqr_kernel<true, false, true>, d_descs, d_eps, C);
    if (C > 1) return cudaLaunchKernelEx(&cfg, hqr_kernel<true, true, true>, d_descs, d_eps, C);
    return cudaLaunchKernelEx(&cfg, hqr_kernel<false, true, true>, d_descs, d_eps, C);
  }
  if (!hqrb_off()) {
    int Cb = 1;
    HqrbSmem Lb;
    if (hqrb_shape(count, max_m, max_nc, &Cb, &Lb)) {
      cfg.gridDim = dim3(count * Cb);
      // >= 120 KB: one CTA per SM (two co-resident clusters would share the SMs' issue slots)
      cfg.dynamicSmemBytes = std::max<size_t>(size_t(Lb.total()) * 8, HQRB_SMEM_MIN);
      attr[0].val.clusterDim.x = Cb;
      cfg.numAttrs = Cb > 1 ? 1 : 0;
      if (std::getenv("DTN_DEBUG_QR"))
        std::fprintf(stderr, "hqrb: cluster %d rmax %d smem %lld\n", Cb, Lb.rmax, Lb.total() * 8);
      if (Cb > 1) return cudaLaunchKernelEx(&cfg, hqrb_kernel<true>, d_descs, d_eps, Cb, Lb);
      return cudaLaunchKernelEx(&cfg, hqrb_kernel<false>, d_descs, d_eps, Cb, Lb);
    }
  }
  if (hqr_legacy()) {
    if (!sm) return cudaLaunchKernelEx(&cfg, hqr_kernel<true, false>, d_descs, d_eps, C);
    if (C > 1) return cudaLaunchKernelEx(&cfg, hqr_kernel<true, true>, d_descs, d_eps, C);
    return cudaLaunchKernelEx(&cfg, hqr_kernel<false, true>, d_descs, d_eps, C);
  }
  if (!sm) return cudaLaunchKernelEx(&cfg, hqr1_kernel<true, false>, d_descs, d_eps, C);
  if (C > 1) return cudaLaunchKernelEx(&cfg, hqr1_kernel<true, true>, d_descs, d_eps, C);
  return cudaLaunchKernelEx(&cfg, hqr1_kernel<false, true>, d_descs, d_eps, C);
}

}  // namespace dtnb
