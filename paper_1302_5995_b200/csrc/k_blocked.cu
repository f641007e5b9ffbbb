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

#include <cooperative_groups.h>

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

// Panel factorisation: GEPP of the panel columns [k0, k0+kbe) over ALL rows
// [k0, total) of the system, pivot search restricted to the interface rows
// [k0, ni) (boundary rows are eliminated but never chosen as pivots). The
// panel lives in registers: a cluster of `csize` CTAs x PNT threads, thread
// owning rows r = rank*PNT + tid + csize*PNT*a. One pivot step = warp argmax
// -> CTA argmax -> (cluster barrier + DSMEM exchange of the candidate rows)
// -> swap + rank-1 update in registers. Also writes ipiv (absolute rows).
namespace cg = cooperative_groups;
constexpr int PNT = 256, PKB = 32, PNW = PNT / 32;

template <int RPT, bool CL>
__global__ void __launch_bounds__(PNT) panel_kernel(KernelArgs args, const int* __restrict__ list, int k0, int kb,
                                                   int csize) {
  __shared__ double wrow[2][PNW][PKB];
  __shared__ double wval[2][PNW];
  __shared__ int wpos[2][PNW];
  __shared__ double cval[2];
  __shared__ int cpos[2], cwarp[2];
  __shared__ double drow[2][PKB];
  __shared__ double prow_s[PKB], jrow_s[PKB];
  __shared__ int s_p;
  const int crank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const int node_id = list[blockIdx.x / csize];
  const NodeDev nd = args.nodes[node_id];
  if (k0 >= nd.ni) return;  // uniform over the cluster
  const int kbe = min(kb, nd.ni - k0);
  const int Ri = nd.ni - k0, Rall = nd.total - k0;
  const int stride = csize * PNT;
  double* M = args.arena + nd.m_off + k0 + (long long)k0 * nd.ldm;
  const long long ldm = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* ipiv = args.piv + nd.piv_off;

  double v[RPT][PKB];
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
#pragma unroll
    for (int c = 0; c < PKB; ++c) v[a][c] = (r < Rall && c < kbe) ? M[r + c * ldm] : 0.0;
  }
  double pmin = k0 == 0 ? DBL_MAX : args.pivstat[2 * node_id];
  double pmax = k0 == 0 ? 0.0 : args.pivstat[2 * node_id + 1];

#pragma unroll
  for (int j = 0; j < PKB; ++j) {
    if (j >= kbe) break;
    const int buf = j & 1;
    // ---- thread / warp argmax over own candidate rows (NaN counts as +inf)
    double best = -1.0;
    int bpos = 0x7fffffff, ba = 0;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
      if (r >= j && r < Ri) {
        double av = fabs(v[a][j]);
        if (av != av) av = INFINITY;
        if (av > best) { best = av; bpos = r; ba = a; }
      }
    }
    double wb = best;
    int wp = bpos;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, wb, off);
      const int op = __shfl_xor_sync(0xffffffffu, wp, off);
      if (ob > wb || (ob == wb && op < wp)) { wb = ob; wp = op; }
    }
    if (wp == bpos && bpos != 0x7fffffff) {  // the owning lane publishes its row
#pragma unroll
      for (int a = 0; a < RPT; ++a)
        if (a == ba) {
#pragma unroll
          for (int c = 0; c < PKB; ++c) wrow[buf][warp][c] = v[a][c];
        }
    }
    if (lane == 0) { wval[buf][warp] = wb; wpos[buf][warp] = wp; }
    {  // the owner of position j publishes row j
      const int rj = j - crank * PNT;
      if (rj >= 0 && (rj % stride) == tid && rj / stride < RPT) {
        const int aj = rj / stride;
#pragma unroll
        for (int a = 0; a < RPT; ++a)
          if (a == aj) {
#pragma unroll
            for (int c = 0; c < PKB; ++c) drow[buf][c] = v[a][c];
          }
      }
    }
    __syncthreads();
    if (warp == 0) {
      double b = lane < PNW ? wval[buf][lane] : -1.0;
      int bp = lane < PNW ? wpos[buf][lane] : 0x7fffffff;
      int bw = lane;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b, off);
        const int op = __shfl_xor_sync(0xffffffffu, bp, off);
        const int ow = __shfl_xor_sync(0xffffffffu, bw, off);
        if (ob > b || (ob == b && op < bp)) { b = ob; bp = op; bw = ow; }
      }
      if (lane == 0) { cval[buf] = b; cpos[buf] = bp; cwarp[buf] = bw; }
    }
    if constexpr (CL) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
    if (warp == 0) {
      double b = -1.0;
      int bp = 0x7fffffff, br = 0, bw = 0;
      if (lane < csize) {
        if constexpr (CL) {
          cg::cluster_group cl = cg::this_cluster();
          b = *cl.map_shared_rank(&cval[buf], lane);
          bp = *cl.map_shared_rank(&cpos[buf], lane);
          bw = *cl.map_shared_rank(&cwarp[buf], lane);
        } else {
          b = cval[buf];
          bp = cpos[buf];
          bw = cwarp[buf];
        }
        br = lane;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {  // all 32 lanes end with the winner
        const double ob = __shfl_xor_sync(0xffffffffu, b, off);
        const int op = __shfl_xor_sync(0xffffffffu, bp, off);
        const int orr = __shfl_xor_sync(0xffffffffu, br, off);
        const int ow = __shfl_xor_sync(0xffffffffu, bw, off);
        if (ob > b || (ob == b && op < bp)) { b = ob; bp = op; br = orr; bw = ow; }
      }
      if (bp == 0x7fffffff) { bp = j; br = (j / PNT) % csize; bw = -1; }  // empty candidate set
      const int rank_j = (j / PNT) % csize;
      if (lane < kbe) {
        if constexpr (CL) {
          cg::cluster_group cl = cg::this_cluster();
          prow_s[lane] = bw >= 0 ? *cl.map_shared_rank(&wrow[buf][bw][lane], br)
                                 : *cl.map_shared_rank(&drow[buf][lane], rank_j);
          jrow_s[lane] = *cl.map_shared_rank(&drow[buf][lane], rank_j);
        } else {
          prow_s[lane] = bw >= 0 ? wrow[buf][bw][lane] : drow[buf][lane];
          jrow_s[lane] = drow[buf][lane];
        }
      }
      if (lane == 0) s_p = bp;
    }
    __syncthreads();
    const int p = s_p;
    const double piv = prow_s[j];
    const double apiv = fabs(piv);
    pmin = fmin(pmin, apiv);
    pmax = (apiv != apiv) ? INFINITY : fmax(pmax, apiv);
    const double rinv = 1.0 / piv;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
      if (r == p && p != j) {
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = jrow_s[c];
      }
      if (r == j) {
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = prow_s[c];
      }
      if (r > j && r < Rall) {
        const double l = v[a][j] * rinv;
        v[a][j] = l;
#pragma unroll
        for (int c = j + 1; c < PKB; ++c) v[a][c] = fma(-l, prow_s[c], v[a][c]);
      }
    }
    if (crank == 0 && tid == 0) ipiv[k0 + j] = k0 + p;
  }
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
    if (r < Rall) {
#pragma unroll
      for (int c = 0; c < PKB; ++c)
        if (c < kbe) M[r + c * ldm] = v[a][c];
    }
  }
  if (crank == 0 && tid == 0) {
    args.pivstat[2 * node_id] = pmin;
    args.pivstat[2 * node_id + 1] = pmax;
  }
  if constexpr (CL) cg::this_cluster().sync();  // keep smem alive for remote readers
}

// Net permutation of the rows touched by the kbe sequential swaps
// (k0+i <-> ipiv[k0+i]): after the swaps, row dst[t] holds old row src[t].
__device__ int panel_permutation(const int* sp, int k0, int kbe, int* dst, int* src) {
  int nt = 0;
  auto find = [&](int row) {
    for (int t = 0; t < nt; ++t)
      if (dst[t] == row) return t;
    dst[nt] = row;
    src[nt] = row;
    return nt++;
  };
  for (int i = 0; i < kbe; ++i) {
    const int a = find(k0 + i), b = find(sp[i]);
    const int t = src[a];
    src[a] = src[b];
    src[b] = t;
  }
  return nt;
}

// Row swaps + U12 = L11^{-1} (P A)[k0:k1, k1:total] for the trailing columns;
// with swap_left, also the row swaps of the already factored columns [0, k0)
// (needed only when L itself is reused: the root LU for G = S^{-1}).
__global__ void __launch_bounds__(RP_THREADS) rowpanel_kernel(KernelArgs args, const int* __restrict__ list, int k0,
                                                              int kb, int ncoltiles, int swap_left) {
  __shared__ double T[32][33];
  __shared__ int s_dst[64], s_src[64], s_piv[32], s_nt;
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  if (k0 >= nd.ni) return;
  const int kbe = min(kb, nd.ni - k0), k1 = k0 + kbe;
  double* M = args.arena + nd.m_off;
  const long long ld = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool left = blockIdx.x >= ncoltiles;
  const int jbase = left ? (blockIdx.x - ncoltiles) * RP_COLS : k1 + blockIdx.x * RP_COLS;
  const int jend = left ? k0 : nd.total;
  if (left && !swap_left) return;
  if (jbase >= jend) return;
  if (tid < kbe) s_piv[tid] = args.piv[nd.piv_off + k0 + tid];
  if (!left)
    for (int e = tid; e < kbe * kbe; e += RP_THREADS) T[e % kbe][e / kbe] = M[(k0 + e % kbe) + (k0 + e / kbe) * ld];
  __syncthreads();
  if (tid == 0) s_nt = panel_permutation(s_piv, k0, kbe, s_dst, s_src);
  __syncthreads();
  const int nt = s_nt;
  for (int jj = warp; jj < RP_COLS; jj += RP_THREADS / 32) {
    const int j = jbase + jj;
    if (j >= jend) break;
    double* col = M + (long long)j * ld;
    const double v0 = lane < nt ? col[s_src[lane]] : 0.0;
    const double v1 = lane + 32 < nt ? col[s_src[lane + 32]] : 0.0;
    __syncwarp();
    if (lane < nt) col[s_dst[lane]] = v0;
    if (lane + 32 < nt) col[s_dst[lane + 32]] = v1;
    __syncwarp();
    if (left) continue;
    double x = lane < kbe ? col[k0 + lane] : 0.0;
    for (int c = 0; c < kbe; ++c) {  // unit lower L11
      const double xc = __shfl_sync(0xffffffffu, x, c);
      if (lane > c && lane < kbe) x = fma(-T[lane][c], xc, x);
    }
    if (lane < kbe) col[k0 + lane] = x;
  }
}

cudaError_t blocked_init() { return cudaSuccess; }

cudaError_t launch_gather(const KernelArgs& args, const int* d_list, int count, int max_total, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((max_total + GATHER_COLS - 1) / GATHER_COLS, count);
  gather_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

// Panel geometry for systems with up to max_rows rows below k0 (kb <= 32).
void panel_shape(int max_rows, int* rpt, int* csize) {
  if (max_rows <= PNT) { *rpt = 1; *csize = 1; return; }
  *rpt = 2;
  *csize = (max_rows + 2 * PNT - 1) / (2 * PNT);
}

template <int RPT, bool CL>
cudaError_t launch_panel_t(const KernelArgs& args, const int* d_list, int count, int k0, int kb, int csize,
                           cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * csize);
  cfg.blockDim = dim3(PNT);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (CL) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, panel_kernel<RPT, CL>, args, d_list, k0, kb, csize);
}

cudaError_t launch_panel(const KernelArgs& args, const int* d_list, int count, int max_rows, int k0, int kb,
                         cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (kb > PKB) return cudaErrorInvalidValue;
  int rpt, csize;
  panel_shape(max_rows, &rpt, &csize);
  if (csize > 8) return cudaErrorInvalidValue;
  if (csize == 1) {
    if (rpt == 1) return launch_panel_t<1, false>(args, d_list, count, k0, kb, 1, st);
    return launch_panel_t<2, false>(args, d_list, count, k0, kb, 1, st);
  }
  return launch_panel_t<2, true>(args, d_list, count, k0, kb, csize, st);
}

cudaError_t launch_rowpanel(const KernelArgs& args, const int* d_list, int count, int max_total, int k0, int kb,
                            bool swap_left, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int coltiles = (max_total - k0 + RP_COLS - 1) / RP_COLS;
  const int lefttiles = swap_left ? (k0 + RP_COLS - 1) / RP_COLS : 0;
  if (coltiles + lefttiles <= 0) return cudaSuccess;
  dim3 grid(coltiles + lefttiles, count);
  rowpanel_kernel<<<grid, RP_THREADS, 0, st>>>(args, d_list, k0, kb, coltiles, swap_left ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace dtnb
