// Blocked merge path for systems too large for one CTA (total > small_max):
//   gather     assemble M = [interface; union boundary]^2 in HBM from the two
//              child Schur complements and the cross-interface couplings
//              (merge_two, dense_nd.cpp:114-165);
//   per panel of kb pivots (right-looking partial LU restricted to the ni
//   interface pivots, partial pivoting among interface rows only —
//   PartialPivLU of M_ii, dense_nd.cpp:174):
//     panel     GEPP of the interface rows of the panel columns, in smem;
//     rowpanel  row swaps + L11^{-1} on the panel rows of the trailing
//               columns (U12), and U11^{-1} on the boundary rows of the
//               panel columns (L21 of the boundary block);
//     trailing  M[k1:,k1:] -= L21 U12 on the DMMA tensor pipe (k_gemm.cu).
// After the last panel the boundary block M[ni:, ni:] holds
// S = M_bb - M_bi M_ii^{-1} M_ib (dense_nd.cpp:181) in place.
#include <cfloat>

#include "common.cuh"

namespace dtnb {

constexpr int GATHER_COLS = 8;
constexpr int PANEL_THREADS = 512;
constexpr int RP_THREADS = 256;
constexpr int RP_COLS = 32;  // trailing columns per rowpanel CTA

__global__ void __launch_bounds__(256) gather_kernel(KernelArgs args, const int* __restrict__ list) {
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  const int j0 = blockIdx.x * GATHER_COLS;
  if (j0 >= nd.total) return;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* A = args.arena + ca.s_off;
  const double* B = args.arena + cb.s_off;
  double* M = args.arena + nd.m_off;
  const PosDev* pos = args.pos + nd.pos_off;
  for (int jj = 0; jj < GATHER_COLS; ++jj) {
    const int j = j0 + jj;
    if (j >= nd.total) break;
    const PosDev pj = pos[j];
    const double* colA = pj.src >= 0 ? A + (long long)pj.src * ca.ld : nullptr;
    const double* colB = pj.src < 0 ? B + (long long)(-pj.src - 1) * cb.ld : nullptr;
    for (int i = threadIdx.x; i < nd.total; i += blockDim.x) {
      const PosDev pi = pos[i];
      double v = 0.0;
      if (pi.src >= 0 && colA) v = colA[pi.src];
      else if (pi.src < 0 && colB) v = colB[-pi.src - 1];
      else if (pi.partner == j) v = args.stencil[pi.dir * args.nu + pi.gid];
      M[i + (long long)j * nd.ldm] = v;
    }
  }
}

// GEPP of the interface rows [k0, ni) x panel columns [k0, k0+kbe), smem-resident.
__global__ void __launch_bounds__(PANEL_THREADS) panel_kernel(KernelArgs args, const int* __restrict__ list, int k0,
                                                              int kb, int node_slot) {
  extern __shared__ double P[];
  __shared__ double s_best[PANEL_THREADS / 32];
  __shared__ int s_idx[PANEL_THREADS / 32];
  __shared__ int s_p;
  const int node_id = list[blockIdx.x + node_slot];
  const NodeDev nd = args.nodes[node_id];
  if (k0 >= nd.ni) return;
  const int kbe = min(kb, nd.ni - k0);
  const int R = nd.ni - k0;
  const int ldp = R | 1;
  double* M = args.arena + nd.m_off + k0 + (long long)k0 * nd.ldm;
  int* ipiv = args.piv + nd.piv_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = 0; c < kbe; ++c)
    for (int r = tid; r < R; r += PANEL_THREADS) P[c * ldp + r] = M[r + (long long)c * nd.ldm];
  __syncthreads();
  double pmin = k0 == 0 ? DBL_MAX : args.pivstat[2 * node_id];
  double pmax = k0 == 0 ? 0.0 : args.pivstat[2 * node_id + 1];
  for (int j = 0; j < kbe; ++j) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = j + tid; r < R; r += PANEL_THREADS) {
      const double av = fabs(P[j * ldp + r]);
      if (av > best) { best = av; bi = r; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { s_best[warp] = best; s_idx[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < PANEL_THREADS / 32 ? s_best[lane] : -1.0;
      bi = lane < PANEL_THREADS / 32 ? s_idx[lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) s_p = bi;
    }
    __syncthreads();
    const int p = s_p;
    if (p != j && tid < kbe) {
      const double t = P[tid * ldp + j];
      P[tid * ldp + j] = P[tid * ldp + p];
      P[tid * ldp + p] = t;
    }
    if (tid == 0) ipiv[k0 + j] = k0 + p;
    __syncthreads();
    const double pv = P[j * ldp + j];
    pmin = fmin(pmin, fabs(pv));
    pmax = fmax(pmax, fabs(pv));
    const double rinv = 1.0 / pv;
    for (int r = j + 1 + tid; r < R; r += PANEL_THREADS) {
      const double l = P[j * ldp + r] * rinv;
      P[j * ldp + r] = l;
      for (int c = j + 1; c < kbe; ++c) P[c * ldp + r] = fma(-l, P[c * ldp + j], P[c * ldp + r]);
    }
    __syncthreads();
  }
  for (int c = 0; c < kbe; ++c)
    for (int r = tid; r < R; r += PANEL_THREADS) M[r + (long long)c * nd.ldm] = P[c * ldp + r];
  if (tid == 0) {
    args.pivstat[2 * node_id] = pmin;
    args.pivstat[2 * node_id + 1] = pmax;
  }
}

// Net permutation of the rows touched by the kbe sequential swaps
// (k0+i <-> ipiv[k0+i]): after the swaps, row dst[t] holds old row src[t].
__device__ int panel_permutation(const int* ipiv, int k0, int kbe, int* dst, int* src) {
  int nt = 0;
  auto find = [&](int row) {
    for (int t = 0; t < nt; ++t)
      if (dst[t] == row) return t;
    dst[nt] = row;
    src[nt] = row;
    return nt++;
  };
  for (int i = 0; i < kbe; ++i) {
    const int a = find(k0 + i), b = find(ipiv[k0 + i]);
    const int t = src[a];
    src[a] = src[b];
    src[b] = t;
  }
  return nt;
}

__global__ void __launch_bounds__(RP_THREADS) rowpanel_kernel(KernelArgs args, const int* __restrict__ list, int k0,
                                                              int kb, int ncoltiles) {
  __shared__ double T[32][33];
  __shared__ int s_dst[64], s_src[64], s_nt;
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  if (k0 >= nd.ni) return;
  const int kbe = min(kb, nd.ni - k0), k1 = k0 + kbe;
  double* M = args.arena + nd.m_off;
  const long long ld = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x < ncoltiles) {
    const int jbase = k1 + blockIdx.x * RP_COLS;
    if (jbase >= nd.total) return;
    for (int e = tid; e < kbe * kbe; e += RP_THREADS) T[e % kbe][e / kbe] = M[(k0 + e % kbe) + (k0 + e / kbe) * ld];
    if (tid == 0) s_nt = panel_permutation(args.piv + nd.piv_off, k0, kbe, s_dst, s_src);
    __syncthreads();
    const int nt = s_nt;
    for (int jj = warp; jj < RP_COLS; jj += RP_THREADS / 32) {
      const int j = jbase + jj;
      if (j >= nd.total) break;
      double* col = M + (long long)j * ld;
      const double v0 = lane < nt ? col[s_src[lane]] : 0.0;
      const double v1 = lane + 32 < nt ? col[s_src[lane + 32]] : 0.0;
      __syncwarp();
      if (lane < nt) col[s_dst[lane]] = v0;
      if (lane + 32 < nt) col[s_dst[lane + 32]] = v1;
      __syncwarp();
      double x = lane < kbe ? col[k0 + lane] : 0.0;
      for (int c = 0; c < kbe; ++c) {  // unit lower L11
        const double xc = __shfl_sync(0xffffffffu, x, c);
        if (lane > c && lane < kbe) x = fma(-T[lane][c], xc, x);
      }
      if (lane < kbe) col[k0 + lane] = x;
    }
  } else {
    const int i = nd.ni + (blockIdx.x - ncoltiles) * RP_THREADS + tid;
    for (int e = tid; e < kbe * kbe; e += RP_THREADS) T[e % kbe][e / kbe] = M[(k0 + e % kbe) + (k0 + e / kbe) * ld];
    __syncthreads();
    if (i >= nd.total) return;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c] = c < kbe ? M[i + (k0 + c) * ld] : 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {  // x <- x U11^{-1}
      if (c < kbe) {
        double s = x[c];
#pragma unroll
        for (int l = 0; l < c; ++l) s = fma(-x[l], T[l][c], s);
        x[c] = s / T[c][c];
      }
    }
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < kbe) M[i + (k0 + c) * ld] = x[c];
  }
}

cudaError_t blocked_init() {
  return cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

cudaError_t launch_gather(const KernelArgs& args, const int* d_list, int count, int max_total, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((max_total + GATHER_COLS - 1) / GATHER_COLS, count);
  gather_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

// kb chosen by the caller so that kb * max_rows * 8 bytes fits in 220 KB.
cudaError_t launch_panel(const KernelArgs& args, const int* d_list, int count, int max_ni, int k0, int kb,
                         cudaStream_t st) {
  if (count <= 0 || k0 >= max_ni) return cudaSuccess;
  const int rows = (max_ni - k0) | 1;
  const size_t smem = size_t(kb) * rows * sizeof(double);
  panel_kernel<<<count, PANEL_THREADS, smem, st>>>(args, d_list, k0, kb, 0);
  return cudaGetLastError();
}

cudaError_t launch_rowpanel(const KernelArgs& args, const int* d_list, int count, int max_total, int min_nb,
                            int max_nb, int k0, int kb, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int coltiles = (max_total - k0 + RP_COLS - 1) / RP_COLS;
  const int rowtiles = (max_nb + RP_THREADS - 1) / RP_THREADS;
  (void)min_nb;
  dim3 grid(coltiles + rowtiles, count);
  rowpanel_kernel<<<grid, RP_THREADS, 0, st>>>(args, d_list, k0, kb, coltiles);
  return cudaGetLastError();
}

}  // namespace dtnb
