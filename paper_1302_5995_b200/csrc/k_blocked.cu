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
#include <cstdlib>
#include <initializer_list>
#include <type_traits>

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
  if (j0 >= nd.ncols) return;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* A = args.arena + ca.s_off;
  const double* B = args.arena + cb.s_off;
  double* M = args.arena + nd.m_off;
  const PosDev* pos = args.pos + nd.pos_off;
  for (int jj = 0; jj < GATHER_COLS; ++jj) {
    const int j = j0 + jj;
    if (j >= nd.ncols) break;
    if (j >= nd.total) {  // body-load column: the children's rhs rows summed into place (dense_nd.cpp:136-146)
      const int c = j - nd.total;
      const double* rA = args.arena + ca.rhs_off + (long long)c * ca.rhs_ld;
      const double* rB = args.arena + cb.rhs_off + (long long)c * cb.rhs_ld;
      for (int i = threadIdx.x; i < nd.total; i += blockDim.x) {
        const PosDev pi = pos[i];
        M[i + (long long)j * nd.ldm] = pi.src >= 0 ? rA[pi.src] : rB[-pi.src - 1];
      }
      continue;
    }
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
// owning rows r = rank*PNT + tid + csize*PNT*a. One pivot step costs one CTA
// barrier and one cluster barrier: each CTA pushes its best candidate row
// (and the owner of row j pushes row j) into every CTA's shared memory with
// remote DSMEM stores before the barrier, so after it the pivot decision and
// the rank-1 update are purely local. Outputs: the factored panel, ipiv
// (absolute rows) and the net row-move list consumed by rowpanel_kernel.
namespace cg = cooperative_groups;
constexpr int PNT = 256, PKB = 32, PNW = PNT / 32, PMAXC = 16;


// ---- DSMEM push with mbarrier completion (no cluster-wide barrier per pivot)
__device__ __forceinline__ unsigned cluster_map(const void* p, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_b64(unsigned addr, unsigned long long v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(v),
               "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_b32(unsigned addr, unsigned v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
               "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v4_b32(unsigned addr, unsigned a, unsigned b, unsigned c, unsigned d,
                                                unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_shared_v2_pred(double* p, double a, double b, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(smem_u32(p)),
               "d"(a), "d"(b), "r"(int(pred))
               : "memory");
}
__device__ __forceinline__ void st_shared_v4u_pred(unsigned* p, unsigned a, unsigned b, unsigned c, unsigned d,
                                                   bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n}" ::"r"(
                   smem_u32(p)),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(int(pred))
               : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// Net row moves of the panel at k0 (64 dst + 64 src slots), double-buffered
// by step parity: the next panel's prologue reads step k0's list while the
// side stream's rowpanel(k0) may still be reading it.
__device__ __forceinline__ int* move_list(const KernelArgs& args, const NodeDev& nd, int k0) {
  return args.piv + nd.piv_off + ((nd.ni + 3) & ~3) + ((k0 / PKB) & 1) * 4 * PKB;
}
// per-node count of panels that needed row interchanges; once it reaches the
// launch's use_fast threshold the no-interchange attempt is skipped for the
// node's remaining panels
__device__ __forceinline__ int* pivoting_flag(const KernelArgs& args, const NodeDev& nd) {
  return args.piv + nd.piv_off + ((nd.ni + 3) & ~3) + 8 * PKB;
}

#ifdef DTN_PANEL_PROFILE
__device__ long long g_panel_clk[8 * 32];
#define PCLK(slot) do { if (blockIdx.x == 0 && tid == 0) g_panel_clk[j * 8 + (slot)] = clock64(); } while (0)
__device__ long long g_pro_clk[8];
#define PROCLK(slot) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_pro_clk[slot] = clock64(); } while (0)
#else
#define PROCLK(slot) do { } while (0)
#endif

#ifdef DTN_PANEL_PROFILE
__device__ long long g_p2_clk[16];
__device__ long long g_p2b_clk[16];  // the same points seen by the LAST thread of the last CTA (a row that works)
#define P2CLK(slot) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_p2_clk[slot] = clock64(); if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x / 2) g_p2b_clk[slot] = clock64(); } while (0)
#define P2ACC(slot, t) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long n_ = clock64(); g_p2_clk[slot] += n_ - (t); (t) = n_; } } while (0)
#else
#define P2CLK(slot) do { } while (0)
#define P2ACC(slot, t) do { } while (0)
#endif

__device__ unsigned g_panel_fallbacks;  // panels whose no-interchange attempt failed (diagnostic)

struct PanelCand {
  unsigned key;
  int pos, lab, pad;
  double row[PKB];
};

// Registers hold one row per thread; the pivot loop is fully unrolled so all
// register indices are compile-time. Rows are NOT swapped during the panel:
// the pivot row of step j is flagged (elim = j) and stays in its thread, so a
// pivot step moves no data except the per-warp candidate rows. The final row
// order (pivot rows to positions [0, kbe), displaced top rows into the
// vacated positions) is applied once at the end, and published as the net
// row-move list + the node's running permutation perm[pos] = original row.
template <bool CL, int RPT>
__global__ void __launch_bounds__(PNT) panel_kernel(KernelArgs args, const int* __restrict__ list, int k0, int kb,
                                                   int csize, int fused, int use_fast) {
  // row slots: [0, PNW) warp candidates, PNW + q = candidate of cluster rank q
  constexpr int SC = PNW, NSLOT = PNW + (CL ? PMAXC : 0);
  __shared__ __align__(16) double rows[2][NSLOT][PKB];
  __shared__ __align__(16) unsigned sinfo[2][PNW][4];  // warp candidates: key, lo, pos
  __shared__ int sp[PKB], vac[PKB];
  __shared__ __align__(16) unsigned cinfo[2][CL ? PMAXC : 1][4];  // cluster candidates: key, lo, pos
  __shared__ __align__(8) unsigned long long mbar[2];
  constexpr int PLD = PKB + 2;  // 16-byte aligned rows
  __shared__ __align__(16) double pro[PKB * PLD];  // prologue: L11 of step k0 - kb, then U12
  __shared__ int m_dst[2 * PKB], m_src[2 * PKB];
  // dynamic: the fast path's U11 rows and reciprocals, and per-thread row
  // storage (the prologue's L21 rows, then the rows saved for a fallback)
  extern __shared__ __align__(16) double pdyn[];
  double* ub = pdyn;                         // [PKB][PLD] rows of U11
  double* urinv = ub + PKB * PLD;            // [PKB] reciprocal pivots
  double* psave = urinv + PKB;               // [RPT * PNT][PKB + 1] rows before the panel
  const int crank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const int node_id = list[blockIdx.x / csize];
  const NodeDev nd = args.nodes[node_id];
  if (k0 >= nd.ni) return;  // uniform over the cluster
  const int kbe = min(kb, nd.ni - k0);
  // interface rows only: the boundary rows' L21 = A_b U11^{-1} is a parallel
  // TRSM done by rowpanel_kernel
  const int Ri = nd.ni - k0;
  double* M = args.arena + nd.m_off + k0 + (long long)k0 * nd.ldm;
  const long long ldm = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int stride = csize * PNT;
  int* perm = args.piv + nd.piv_off;  // running permutation of the interface rows

  double v[RPT][PKB];
  int elim[RPT];
  // no-interchange attempt for this panel? (every CTA reads the node's count
  // before any can pass the cluster barriers ahead of a fallback that bumps
  // it; k0 == 0 starts clean)
  const bool try_fast = use_fast && (k0 == 0 || *(volatile int*)pivoting_flag(args, nd) < use_fast);
  if (k0 == 0 && crank == 0 && tid == 0) *pivoting_flag(args, nd) = 0;
  if (k0 == 0 || !fused) {
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;  // original panel row
#pragma unroll
      for (int c = 0; c < PKB; ++c) v[a][c] = (r < Ri && c < kbe) ? M[r + c * ldm] : 0.0;
      if (k0 == 0 && r < Ri) perm[r] = r;
    }
  } else {
    // ---- fused prologue: step kp = k0 - kb is applied to this panel's
    // columns here -- its row moves, U12 = L11^{-1} (P A)[kp:k0, cols] and the
    // rank-kb update with L21 -- so the panel chain never waits for the
    // rowpanel / trailing kernels, which handle the other columns of step kp
    // on the side stream concurrently with this panel.
    const int kp = k0 - kb;  // step kp was a full-width step (k0 < ni)
    PROCLK(0);
    double* Mg = args.arena + nd.m_off;  // absolute indexing
    // issue every load up front: this thread's L21 rows (into its row
    // storage) and L11 (into ub, free until the fast path) by cp.async, its
    // rows of the panel columns speculatively from the unmoved position, the
    // move list
    double* l11 = ub;  // [PKB][PLD], L11[i][m] at i * PLD + m
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
      double* lr = psave + (a * PNT + tid) * (PKB + 1);
      if (r < Ri) {
        const long long R = k0 + r;
        for (int m = 0; m < kb; ++m) cp_async8(lr + m, Mg + R + (long long)(kp + m) * ldm, 8);
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = c < kbe ? Mg[R + (long long)(k0 + c) * ldm] : 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = 0.0;
      }
    }
    for (int e = tid; e < PKB * PKB; e += PNT) {
      const int i = e % PKB, m = e / PKB;
      if (m < i && i < kb) cp_async8(l11 + i * PLD + m, Mg + (kp + i) + (long long)(kp + m) * ldm, 8);
      else l11[i * PLD + m] = 0.0;
    }
    cp_async_commit();
    const int* mvp = move_list(args, nd, kp);
    if (tid < 2 * PKB) {
      m_dst[tid] = mvp[tid];
      m_src[tid] = mvp[2 * PKB + tid];
    }
    // U12 right-hand sides (the top rows moved by step kp; warp w solves
    // columns 4w..4w+3 with lane = row), loaded speculatively from the
    // unmoved rows and reloaded below only if step kp interchanged
    constexpr int QC = PKB / PNW;  // columns per warp
    double xs[QC];
#pragma unroll
    for (int q = 0; q < QC; ++q)
      xs[q] = (lane < kb && warp * QC + q < kbe) ? Mg[(kp + lane) + (long long)(k0 + warp * QC + q) * ldm] : 0.0;
    cp_async_wait<0>();
    __syncthreads();
    PROCLK(1);
    // U12 = L11^{-1} (moved top rows) by all warps: warp w solves columns
    // 4w..4w+3 with lane = row (slot i moves a row into kp + i), the solved
    // entry of row m broadcast by shuffle at step m
    {
      const int i = lane, c0 = warp * QC;
      const int srow = m_src[i];
      double x[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q)
        x[q] = (srow == kp + i || !(i < kb && c0 + q < kbe)) ? xs[q] : Mg[srow + (long long)(k0 + c0 + q) * ldm];
#pragma unroll 4
      for (int m = 0; m < kb - 1; ++m) {
        const double lim = (i > m) ? l11[i * PLD + m] : 0.0;
#pragma unroll
        for (int q = 0; q < QC; ++q) x[q] = fma(-lim, __shfl_sync(0xffffffffu, x[q], m), x[q]);
      }
#pragma unroll
      for (int q = 0; q < QC; ++q) pro[i * PLD + c0 + q] = x[q];  // U12[i][c]; written to M after the loop
    }
    // rows displaced by step kp's interchanges (rare) reload from their source
    const bool displaced = m_dst[PKB] >= 0;  // slots >= PKB list rows moved below the top block
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
      if (displaced && r < Ri) {
        const int R = k0 + r;
        int src = R;
#pragma unroll 4
        for (int t = PKB; t < 2 * PKB; ++t)  // vacated positions (>= kp + kb)
          if (m_dst[t] == R) src = m_src[t];
        if (src != R)
#pragma unroll
          for (int c = 0; c < PKB; ++c) v[a][c] = c < kbe ? Mg[src + (long long)(k0 + c) * ldm] : 0.0;
      }
    }
    __syncthreads();
    PROCLK(2);
    // the fast path's top-block LU (warp 0 of rank 0) waits only for warp 0's
    // own rows: the other warps of that CTA update theirs while it factors
    const bool lead = try_fast && crank == 0;
    if (lead && warp != 0) asm volatile("bar.sync 1, %0;" ::"r"(PNT) : "memory");
    // rank-kb update with L21, rolled over m (the unrolled 1024-FMA form ran
    // at the instruction-fetch rate)
#pragma unroll 2
    for (int m = 0; m < kb; ++m) {
      double lm[RPT];
#pragma unroll
      for (int a = 0; a < RPT; ++a) lm[a] = psave[(a * PNT + tid) * (PKB + 1) + m];
      const double2* u2 = reinterpret_cast<const double2*>(pro + m * PLD);
#pragma unroll
      for (int c2 = 0; c2 < PKB / 2; ++c2) {
        const double2 u = u2[c2];
#pragma unroll
        for (int a = 0; a < RPT; ++a) {
          v[a][2 * c2] = fma(-lm[a], u.x, v[a][2 * c2]);
          v[a][2 * c2 + 1] = fma(-lm[a], u.y, v[a][2 * c2 + 1]);
        }
      }
    }
    if (lead && warp == 0) asm volatile("bar.arrive 1, %0;" ::"r"(PNT) : "memory");
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
#pragma unroll
      for (int c = 0; c < PKB; ++c)
        if (c >= kbe || r >= Ri) v[a][c] = 0.0;
    }
  }
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
    elim[a] = (r < Ri) ? -1 : PKB;  // step at which this row became a pivot
  }
  PROCLK(3);
  double pmin = k0 == 0 ? DBL_MAX : args.pivstat[2 * node_id];
  double pmax = k0 == 0 ? 0.0 : args.pivstat[2 * node_id + 1];
  bool bad = false;
  // ---- fast path: the panel without row interchanges, verified. Partial
  // pivoting keeps the diagonal whenever no entry below it is larger in
  // magnitude, i.e. whenever every multiplier satisfies |l| <= 1 (ties resolve
  // to the lowest row, the diagonal); the merge and root systems of these
  // operators almost never interchange (config-2 root: 3 of 2044 steps). So
  // the top kbe x kbe block is factored by one warp, every other row solves
  // x U11 = a with the same operation order as the right-looking elimination
  // (bit-identical to the pivoted path), and if any |l| > 1 (or non-finite)
  // anywhere in the panel, the panel is redone from the saved rows by the
  // pivoted loop below -- the result is always that of partial pivoting.
  __shared__ int fast_fail;
  bool fast = false;
  int jstart = 0;  // the pivoted loop resumes here: steps < jstart needed no interchange
  __shared__ int jtop_s, fail_all;
  if (try_fast) {
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
      for (int c = 0; c < PKB; ++c) psave[(a * PNT + tid) * (PKB + 1) + c] = v[a][c];
    if (tid == 0) fast_fail = fail_all = PKB;  // first step needing an interchange (PKB: none)
    int jf = PKB;
    PROCLK(4);
    if (crank == 0 && warp == 0) {  // rows 0..kbe-1 live in lanes 0..kbe-1 (a = 0)
#pragma unroll
      for (int j = 0; j < PKB; ++j) {
        if (j < kbe) {
          const double pj = __shfl_sync(0xffffffffu, v[0][j], j);
          double pr[PKB];
#pragma unroll
          for (int c = j + 1; c < PKB; ++c) pr[c] = __shfl_sync(0xffffffffu, v[0][c], j);
          const double rinv = __drcp_rn(pj);
          if (lane == j) urinv[j] = rinv;
          if (lane > j && lane < kbe) {
            const double l = v[0][j] * rinv;
            v[0][j] = l;
            if (!(fabs(l) <= 1.0) && jf == PKB) jf = j;
#pragma unroll
            for (int c = j + 1; c < PKB; ++c) v[0][c] = fma(-l, pr[c], v[0][c]);
          }
        }
      }
      // U11 rows for the substitution (row-major, 16-byte aligned)
#pragma unroll
      for (int c = 0; c < PKB; ++c) ub[lane * PLD + c] = (c >= lane) ? v[0][c] : 0.0;
      const int jt = __reduce_min_sync(0xffffffffu, unsigned(jf));
      if (lane == 0) fast_fail = jt;
    }
    if constexpr (CL) {
      cg::this_cluster().sync();  // rank 0's U11 and first failing step complete
      if (crank != 0) {
        const double* rub = cg::this_cluster().map_shared_rank(ub, 0);
        for (int e = tid; e < PKB * PLD + PKB; e += PNT) ub[e] = rub[e];
        if (tid == 0) jtop_s = *cg::this_cluster().map_shared_rank(&fast_fail, 0);
      }
    }
    __syncthreads();
    if (crank == 0 && tid == 0) jtop_s = fast_fail;
    __syncthreads();
    const int jtop = jtop_s;  // every row below fails no later than the top block
    PROCLK(5);
    // every row below the top block: x U11 = a (forward substitution), the
    // elimination's own operation order, steps < jmax
    auto subst = [&](int rlo, int jmax, bool track) {
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = crank * PNT + tid + stride * a;
        if (r >= rlo && r < Ri) {
#pragma unroll
          for (int j = 0; j < PKB; ++j) {
            if (j < jmax) {
              const double l = v[a][j] * urinv[j];
              v[a][j] = l;
              if (track && !(fabs(l) <= 1.0) && jf == PKB) jf = j;
              if ((j + 1) & 1) v[a][j + 1] = fma(-l, ub[j * PLD + j + 1], v[a][j + 1]);
#pragma unroll
              for (int c = (j + 2) & ~1; c < PKB; c += 2) {
                const double2 u2 = *reinterpret_cast<const double2*>(&ub[j * PLD + c]);
                v[a][c] = fma(-l, u2.x, v[a][c]);
                v[a][c + 1] = fma(-l, u2.y, v[a][c + 1]);
              }
            }
          }
        }
      }
    };
    subst(kbe, min(kbe, jtop), true);
    // first failing step over the panel (every CTA of the cluster)
    if (jf < PKB) atomicMin(&fast_fail, jf);
    __syncthreads();
    PROCLK(6);
    int jstar;
    if constexpr (CL) {
      // every CTA folds its minimum into every CTA's copy: one cluster barrier
      if (warp == 0 && lane < csize && fast_fail < PKB)
        atomicMin(cg::this_cluster().map_shared_rank(&fail_all, lane), fast_fail);
      cg::this_cluster().sync();
      jstar = fail_all;
    } else {
      jstar = fast_fail;
    }
    jstar = min(jstar, kbe);
    fast = jstar >= kbe;
    PROCLK(7);
    // pivot statistics of the pivots taken without interchanges (rank 0 warp 0 owns them)
    if (crank == 0 && warp == 0) {
      const double apiv = fabs(ub[lane * PLD + lane]);
      const bool live = lane < jstar;
      double lo = live ? apiv : DBL_MAX, hi = live ? apiv : 0.0;
      const bool nb_ = live && (!(apiv == apiv) || apiv == INFINITY);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      pmin = fmin(pmin, lo);
      pmax = fmax(pmax, hi);
      bad |= __any_sync(0xffffffffu, nb_);
    }
    if (fast) {
      // identity placement; the move list moves every pivot row onto itself
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = crank * PNT + tid + stride * a;
        if (r < Ri)
#pragma unroll
          for (int c = 0; c < PKB; ++c)
            if (c < kbe) M[r + c * ldm] = v[a][c];
      }
      if (crank == 0 && tid < 2 * PKB) {
        int* mv = move_list(args, nd, k0);
        mv[tid] = tid < kbe ? k0 + tid : -1;
        mv[2 * PKB + tid] = tid < kbe ? k0 + tid : -1;
      }
    } else {
      // steps < jstar are exactly those of partial pivoting (no interchange):
      // rows >= jstar restart from the saved values with only those steps, rows
      // < jstar (the top LU's lanes) are the pivot rows of steps 0..jstar-1
      if (crank == 0 && tid == 0) {
        atomicAdd(&g_panel_fallbacks, 1u);
        *pivoting_flag(args, nd) += 1;
      }
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = crank * PNT + tid + stride * a;
        if (r >= jstar)
#pragma unroll
          for (int c = 0; c < PKB; ++c) v[a][c] = psave[(a * PNT + tid) * (PKB + 1) + c];
      }
      subst(jstar, jstar, false);
      jstart = jstar;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = crank * PNT + tid + stride * a;
        if (r < jstart) elim[a] = r;
      }
      if (tid < jstart) sp[tid] = tid;
    }
  }
  if (!fast) {
  // every CTA receives csize candidates per pivot: 32 row doubles + key, lo, pos
  const unsigned tx_bytes = unsigned(csize) * (PKB * 8 + 16);
  if constexpr (CL) {
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(&mbar[0], tx_bytes);
      mbar_arm(&mbar[1], tx_bytes);
    }
    cg::this_cluster().sync();  // all barriers armed before any push
  }

#pragma unroll
  for (int j = 0; j < PKB; ++j) {
    if (j >= kbe) break;
    if (j < jstart) continue;
#ifdef DTN_PANEL_PROFILE
    PCLK(0);
#endif
    const int jr = j - jstart;  // mbarrier phases count the executed steps
    const int buf = jr & 1;
    // ---- argmax of |column j| over the live rows: 32-bit key = high word of
    // |x| (sign 0, exponent, 20 mantissa bits; NaN ranks highest), low bit
    // set for candidates; hardware warp max + ballot, ties -> lowest lane
    // exact argmax: max of the high words, then of the low words among the
    // lanes holding that high word (|x| >= 0 orders like its bit pattern)
    unsigned key = 0u, klo = 0u;
    int ba = 0;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const double ax = fabs(v[a][j]);
      const unsigned ka = elim[a] < 0 ? (unsigned(__double2hiint(ax)) | 0x80000000u) : 0u;
      const unsigned kl = unsigned(__double2loint(ax));
      if (ka > key || (ka == key && kl > klo)) { key = ka; klo = kl; ba = a; }
    }
    const unsigned whi = __reduce_max_sync(0xffffffffu, key);
    const unsigned wlo = __reduce_max_sync(0xffffffffu, key == whi ? klo : 0u);
    const int wlane = __ffs(__ballot_sync(0xffffffffu, key == whi && klo == wlo)) - 1;
    const unsigned wkey = whi;
#ifdef DTN_PANEL_PROFILE
    PCLK(1);
#endif
#ifdef DTN_PUBLISH_BRANCH
    if (lane == wlane) {
#pragma unroll
      for (int a = 0; a < RPT; ++a)
        if (a == ba) {
#pragma unroll
          for (int c = j; c < PKB; ++c) rows[buf][warp][c] = v[a][c];
        }
      sinfo[buf][warp][0] = wkey;
      sinfo[buf][warp][1] = wlo;
      sinfo[buf][warp][2] = unsigned(crank * PNT + tid + stride * ba);
    }
#else
    // branch-free publish: predicated shared stores by the winning lane (a
    // divergent branch here cost several hundred cycles per pivot)
    {
      const bool win = lane == wlane;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const bool wa = win && a == ba;
#pragma unroll
        for (int c = j & ~1; c < PKB; c += 2) st_shared_v2_pred(&rows[buf][warp][c], v[a][c], v[a][c + 1], wa);
      }
      st_shared_v4u_pred(&sinfo[buf][warp][0], wkey, wlo, unsigned(crank * PNT + tid + stride * ba), 0u, win);
    }
#endif
#ifdef DTN_PANEL_PROFILE
    PCLK(2);
#endif
    __syncthreads();
#ifdef DTN_PANEL_PROFILE
    PCLK(3);
#endif
    // ---- CTA argmax (every warp, redundantly)
    const unsigned lk = lane < PNW ? sinfo[buf][lane][0] : 0u;
    const unsigned ll = lane < PNW ? sinfo[buf][lane][1] : 0u;
    const unsigned bkey = __reduce_max_sync(0xffffffffu, lk);
    const unsigned blo = __reduce_max_sync(0xffffffffu, lk == bkey ? ll : 0u);
    const int bw = __ffs(__ballot_sync(0xffffffffu, lk == bkey && ll == blo && lane < PNW)) - 1;
    int slot = bw, p = int(sinfo[buf][bw][2]);
    if constexpr (CL) {
      // warp 0 pushes this CTA's candidate into slot SC+crank of every CTA
      // with st.async; each CTA waits on its own mbarrier for all csize
      // candidates (no cluster-wide barrier on the critical path)
      // (warp w serves destinations w, w + PNW: the push is not serialised
      // in one warp; key, lo and pos travel as one 16-byte store)
      {
        const double rv = rows[buf][bw][lane];
        for (int d = warp; d < csize; d += PNW) {
          const unsigned mb = cluster_map(&mbar[buf], d);
          st_async_b64(cluster_map(&rows[buf][SC + crank][lane], d), __double_as_longlong(rv), mb);
          if (lane == 0) st_async_v4_b32(cluster_map(&cinfo[buf][crank][0], d), bkey, blo, unsigned(p), 0u, mb);
        }
      }
      mbar_wait(&mbar[buf], unsigned(jr >> 1) & 1u);
      const unsigned ck = lane < csize ? cinfo[buf][lane][0] : 0u;
      const unsigned cl_ = lane < csize ? cinfo[buf][lane][1] : 0u;
      const unsigned gkey = __reduce_max_sync(0xffffffffu, ck);
      const unsigned glo = __reduce_max_sync(0xffffffffu, ck == gkey ? cl_ : 0u);
      const int cw = __ffs(__ballot_sync(0xffffffffu, ck == gkey && cl_ == glo && lane < csize)) - 1;
      slot = SC + cw;
      p = int(cinfo[buf][cw][2]);
    }
#ifdef DTN_PANEL_PROFILE
    PCLK(4);
#endif
    double pr[PKB];
#pragma unroll
    for (int c = j; c < PKB; ++c) pr[c] = rows[buf][slot][c];
    if constexpr (CL) {
      // re-arm for column j + 2: remote pushes for j + 2 can only start after
      // this CTA's own column j + 1 push, i.e. after this column is consumed
      if (tid == 0) mbar_arm(&mbar[buf], tx_bytes);
    }
    const double piv = pr[j];
    const double apiv = fabs(piv);
    pmin = fmin(pmin, apiv);
    pmax = fmax(pmax, apiv);
    bad |= !(apiv == apiv) || apiv == INFINITY;
    const double rinv = __drcp_rn(piv);
#ifdef DTN_PANEL_PROFILE
    PCLK(5);
#endif
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = crank * PNT + tid + stride * a;
      if (r == p) elim[a] = j;
      if (elim[a] < 0) {
        const double l = v[a][j] * rinv;
        v[a][j] = l;
#pragma unroll
        for (int c = j + 1; c < PKB; ++c) v[a][c] = fma(-l, pr[c], v[a][c]);
      }
    }
#ifdef DTN_PANEL_PROFILE
    PCLK(6);
#endif
    if (tid == 0) sp[j] = p;
#ifdef DTN_PANEL_PROFILE
    PCLK(7);
#endif
  }
  __syncthreads();
  // ---- final placement: pivot of step e -> position e; the top rows [0, kbe)
  // that were not pivots fill, in order, the positions vacated by pivots that
  // came from rows >= kbe (also in order)
  if (warp == 0) {
    const int x = lane < kbe ? sp[lane] : 0x7fffffff;
    const int key2 = x >= kbe ? x : 0x7fffffff;
    int rank = 0;
    for (int e = 0; e < kbe; ++e) {
      const int y = sp[e] >= kbe ? sp[e] : 0x7fffffff;
      rank += (y < key2);
    }
    if (lane < kbe && key2 != 0x7fffffff) vac[rank] = key2;
  }
  unsigned topmask = 0u;  // top rows [0, kbe) that became pivots
#pragma unroll
  for (int e = 0; e < PKB; ++e)
    if (e < kbe && sp[e] < kbe) topmask |= 1u << sp[e];
  __syncthreads();
  int* mv = move_list(args, nd, k0);
  int fp[RPT];
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
    fp[a] = r;
    if (elim[a] >= 0 && elim[a] < PKB) fp[a] = elim[a];
    else if (r < kbe) fp[a] = vac[__popc(~topmask & ((1u << r) - 1u))];  // displaced top row
    if (r < Ri) {
#pragma unroll
      for (int c = 0; c < PKB; ++c)
        if (c < kbe) M[fp[a] + c * ldm] = v[a][c];
      int slot = -1;
      if (fp[a] < kbe) slot = fp[a];
      else if (fp[a] != r) {  // a vacated position: its rank among them
        int rk = 0;
        for (int e = 0; e < kbe; ++e) rk += (sp[e] >= kbe && sp[e] < fp[a]);
        slot = kbe + rk;
      }
      if (slot >= 0) {
        mv[slot] = k0 + fp[a];
        mv[2 * PKB + slot] = k0 + r;
      }
    }
  }
  if (crank == 0) {
    const int nvac = __popc(~topmask & ((kbe < 32) ? ((1u << kbe) - 1u) : 0xffffffffu));
    if (tid >= kbe + nvac && tid < 2 * PKB) {
      mv[tid] = -1;
      mv[2 * PKB + tid] = -1;
    }
  }
  // running permutation: perm[k0 + fp] = old perm[k0 + r] for the moved rows
  if constexpr (CL) cg::this_cluster().sync();
  else __syncthreads();
  int oldp[RPT];
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
    oldp[a] = (r < Ri && fp[a] != r) ? perm[k0 + r] : 0;
  }
  if constexpr (CL) cg::this_cluster().sync();
  else __syncthreads();
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = crank * PNT + tid + stride * a;
    if (r < Ri && fp[a] != r) perm[k0 + fp[a]] = oldp[a];
  }
  }
  if (fused && k0 > 0 && crank == 0) {  // U12 of the prologue into rows [k0 - kb, k0)
    double* Mg = args.arena + nd.m_off;
    for (int e = tid; e < PKB * PKB; e += PNT) {
      const int i = e % PKB, c = e / PKB;
      if (i < kb && c < kbe) Mg[(k0 - kb + i) + (long long)(k0 + c) * ldm] = pro[i * PLD + c];
    }
  }
  if (crank == 0 && tid == 0) {
    args.pivstat[2 * node_id] = pmin;
    args.pivstat[2 * node_id + 1] = bad ? INFINITY : pmax;
  }
  if constexpr (CL) cg::this_cluster().sync();  // no CTA exits while others may still write its smem
}

// ---------------------------------------------------------------------------
// panel2_kernel: panel_kernel's contract and arithmetic (bit-identical results),
// loop-ROLLED. panel_kernel unrolls all 32 pivot steps over compile-time register
// indices (26k SASS instructions, ~415 KB of code executed once per launch: the
// launch is instruction-fetch bound, ncu "no_instructions" stalls). Here every
// row lives in a SHIFTING register window: at step j, w[c] holds column j + c,
// so the step body is the same for every j -- the pivot column is always w[0]
// and the update w[c - 1] = w[c] - l u[c] shifts the window by one -- and the
// step loop is rolled (a few KB of code, icache-resident). Multipliers leave the
// window at their step and go straight to global memory (column-major: a warp's
// stores are coalesced); a pivot row writes its U row when it is chosen. The
// final row placement moves only the <= 2 kb rows that change position (rank 0,
// staged through shared memory after a cluster barrier).
__device__ __forceinline__ void shift_update(double (&w)[PKB], double l, const double* __restrict__ prow) {
  const double2* p2 = reinterpret_cast<const double2*>(prow);
#pragma unroll
  for (int c2 = 0; c2 < PKB / 2; ++c2) {
    const double2 u = p2[c2];
    if (c2 > 0) w[2 * c2 - 1] = fma(-l, u.x, w[2 * c2]);
    w[2 * c2] = fma(-l, u.y, w[2 * c2 + 1]);
  }
  w[PKB - 1] = 0.0;
}

// the same step on a window of W live entries (steps j >= 32 - W: columns past the
// panel are zero, so only w[0 .. W) can change)
template <int W>
__device__ __forceinline__ void shift_update_w(double (&w)[PKB], double l, const double* __restrict__ prow) {
  const double2* p2 = reinterpret_cast<const double2*>(prow);
#pragma unroll
  for (int c2 = 0; c2 < W / 2; ++c2) {
    const double2 u = p2[c2];
    if (c2 > 0) w[2 * c2 - 1] = fma(-l, u.x, w[2 * c2]);
    w[2 * c2] = fma(-l, u.y, w[2 * c2 + 1]);
  }
  w[W - 1] = 0.0;
}
template <int W>
using WinC = std::integral_constant<int, W>;

// Final row placement of a factored panel (whole CTA): pivot of step e -> position e; the
// top rows [0, kbe) that were not pivots fill, in order, the positions vacated by pivots
// from below (also in order). Writes the U rows from ub (shifted), the net move list mv
// and the moved rows' permutation entries; stage holds 2 PKB x PKB doubles.
template <int NTH>
__device__ void place_panel_rows(double* __restrict__ M, long long ldm, int k0, int kbe, const int* sp, int* vac,
                                 int* mv_dst, int* mv_src, const double* ub, double* stage, int* perm, int* mv) {
  constexpr int PNT = NTH, PLD = PKB + 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // U row e (ub, shifted) into the pivot row's original position, columns [e, kbe)
  for (int e = tid; e < PKB * PKB; e += PNT) {
    const int i = e % PKB, c = e / PKB;
    if (i < kbe && c >= i && c < kbe) M[sp[i] + (long long)c * ldm] = ub[i * PLD + (c - i)];
  }
  __syncthreads();
  if (warp == 0) {
    const int x = lane < kbe ? sp[lane] : 0x7fffffff;
    const int key2 = x >= kbe ? x : 0x7fffffff;
    int rk = 0;
    for (int e = 0; e < kbe; ++e) {
      const int y = sp[e] >= kbe ? sp[e] : 0x7fffffff;
      rk += (y < key2);
    }
    if (lane < kbe && key2 != 0x7fffffff) vac[rk] = key2;
    unsigned topmask = 0u;
    for (int e = 0; e < kbe; ++e)
      if (sp[e] < kbe) topmask |= 1u << sp[e];
    __syncwarp();
    // slots: e < kbe -> (dst e, src sp[e]); kbe + i -> (dst vac[i], src i-th displaced top row)
    for (int sl = lane; sl < 2 * PKB; sl += 32) {
      int dst = -1, src = -1;
      if (sl < kbe) {
        dst = sl;
        src = sp[sl];
      } else {
        const int i = sl - kbe;
        const int nvac = __popc(~topmask & ((kbe < 32) ? ((1u << kbe) - 1u) : 0xffffffffu));
        if (i < nvac) {
          // the i-th top row (ascending) that is not a pivot
          int t = 0, cnt = -1;
          for (; t < kbe; ++t)
            if (!((topmask >> t) & 1u) && ++cnt == i) break;
          dst = vac[i];
          src = t;
        }
      }
      mv_dst[sl] = dst;
      mv_src[sl] = src;
    }
  }
  __syncthreads();
  if (tid < 2 * PKB) {
    mv[tid] = mv_dst[tid] >= 0 ? k0 + mv_dst[tid] : -1;
    mv[2 * PKB + tid] = mv_src[tid] >= 0 ? k0 + mv_src[tid] : -1;
  }
  // stage the moved rows (panel columns) and their permutation entries
  for (int e = tid; e < 2 * PKB * PKB; e += PNT) {
    const int sl = e / PKB, c = e % PKB;
    const int src = mv_src[sl];
    if (src >= 0 && mv_dst[sl] != src && c < kbe) stage[sl * PKB + c] = __ldcg(M + src + (long long)c * ldm);
  }
  int oldp = 0;
  if (tid < 2 * PKB && mv_src[tid] >= 0 && mv_dst[tid] != mv_src[tid]) oldp = __ldcg(perm + k0 + mv_src[tid]);
  __syncthreads();
  for (int e = tid; e < 2 * PKB * PKB; e += PNT) {
    const int sl = e / PKB, c = e % PKB;
    const int src = mv_src[sl];
    if (src >= 0 && mv_dst[sl] != src && c < kbe) M[mv_dst[sl] + (long long)c * ldm] = stage[sl * PKB + c];
  }
  if (tid < 2 * PKB && mv_src[tid] >= 0 && mv_dst[tid] != mv_src[tid]) perm[k0 + mv_dst[tid]] = oldp;
}

template <bool CL, int RPT, int NT = PNT>
__global__ void __launch_bounds__(NT) panel2_kernel(KernelArgs args, const int* __restrict__ list, int k0, int kb,
                                                   int csize, int fused, int use_fast) {
  // NT threads per CTA (one row each per RPT): 128-thread CTAs put a 2048-row panel on 16
  // SMs instead of 8, halving each CTA's prologue update and substitution
  constexpr int PNT = NT, PNW = NT / 32;
  constexpr int SC = PNW, NSLOT = PNW + (CL ? PMAXC : 0);
  __shared__ __align__(16) double rows[2][NSLOT][PKB];
  __shared__ __align__(16) unsigned sinfo[2][PNW][4];
  __shared__ int sp[PKB], vac[PKB];
  __shared__ __align__(16) unsigned cinfo[2][CL ? PMAXC : 1][4];
  __shared__ __align__(8) unsigned long long mbar[2];
  constexpr int PLD = PKB + 2;  // 16-byte aligned rows
  __shared__ __align__(16) double pro[PKB * PLD];  // prologue: U12 of step k0 - kb
  __shared__ int m_dst[2 * PKB], m_src[2 * PKB];
  __shared__ int fast_fail, jtop_s, fail_all;
  __shared__ int mv_dst[2 * PKB], mv_src[2 * PKB];
  __shared__ __align__(8) unsigned long long mbar_u[PKB];  // pipelined substitution: one per U row
  extern __shared__ __align__(16) double pdyn[];
  double* ub = pdyn;               // [PKB][PLD]: U11 rows SHIFTED, ub[j * PLD + c] = U[j][j + c]
  double* urinv = ub + PKB * PLD;  // [PKB] reciprocal pivots
  double* psave = urinv + PKB;     // [RPT * PNT][PKB + 1]: L21 rows (prologue), rows before the panel
  const int crank = CL ? int(cg::this_cluster().block_rank()) : 0;
  const int node_id = list[blockIdx.x / csize];
  const NodeDev nd = args.nodes[node_id];
  if (k0 >= nd.ni) return;  // uniform over the cluster
  const int kbe = min(kb, nd.ni - k0);
  const int Ri = nd.ni - k0;
  double* M = args.arena + nd.m_off + k0 + (long long)k0 * nd.ldm;
  const long long ldm = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int stride = csize * PNT;
  int* perm = args.piv + nd.piv_off;
  auto csync = [] {
    if constexpr (CL) cg::this_cluster().sync();
    else __syncthreads();
  };

  P2CLK(0);
  double v[RPT][PKB];
  int elim[RPT];
  const bool pipe_req = (use_fast & 0x20000000) != 0;  // launcher flag (DTN_PANEL_PIPE)
  use_fast &= ~0x20000000;
  const bool try_fast = use_fast && (k0 == 0 || *(volatile int*)pivoting_flag(args, nd) < use_fast);
  if (k0 == 0 && crank == 0 && tid == 0) *pivoting_flag(args, nd) = 0;
  // Pipelined substitution (clusters): rank 0's warp 0 pushes every U row of the top block to all
  // CTAs as it is formed (st.async + one mbarrier per row), and the rows below run substitution
  // step j as soon as row j has landed -- they trail the top LU by one step instead of
  // starting after it.
  // (pipelined launches use the LIGHT LEAD row map: rank 0 holds only the 32 top rows, so its warp 0
  // factors the top block with no other warp of its SM computing; warp 1 forwards the rows)
  const bool lead32 = CL && pipe_req;
  const bool piped = lead32 && try_fast;
  auto rowof = [&](int a_) -> int {
    if (!lead32) return crank * PNT + tid + stride * a_;
    if (crank == 0) return (a_ == 0 && tid < PKB) ? tid : (1 << 28);
    return PKB + (crank - 1) * PNT + tid + (csize - 1) * PNT * a_;
  };
  const bool idle_warp = lead32 && crank == 0 && warp != 0;  // no rows: skips the prologue update
  if constexpr (CL) {
    if (piped) {
      if (tid == 0) fast_fail = fail_all = PKB;
      if (tid < PKB) mbar_init(&mbar_u[tid], 1);
      if (tid < PKB) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      __syncthreads();
      if (tid < kbe && crank != 0) mbar_arm(&mbar_u[tid], (PKB + 1) * 8);  // (rank 0: a plain arrive by warp 0)
      cg::this_cluster().sync();  // every CTA's barriers are armed before the first push
    }
  }
  if (k0 == 0 || !fused) {
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = rowof(a);
#pragma unroll
      for (int c = 0; c < PKB; ++c) v[a][c] = (r < Ri && c < kbe) ? M[r + c * ldm] : 0.0;
      if (k0 == 0 && r < Ri) perm[r] = r;
    }
  } else {
    // fused prologue (as panel_kernel): step kp = k0 - kb applied to this panel's columns
    const int kp = k0 - kb;
    double* Mg = args.arena + nd.m_off;
    // [PKB][PLD], L11[i][m] at i * PLD + m (unshifted). ub is free until the fast path -- unless rows
    // are pushed into it by rank 0 while this CTA is still here (pipelined): then the pivoted loop's
    // exchange buffer, idle until that loop, holds it
    double* l11 = piped ? &rows[0][0][0] : ub;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = rowof(a);
      double* lr = psave + (a * PNT + tid) * (PKB + 1);
      if (r < Ri) {
        const long long R = k0 + r;
        for (int m = 0; m < kb; ++m) cp_async8(lr + m, Mg + R + (long long)(kp + m) * ldm, 8);
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = c < kbe ? Mg[R + (long long)(k0 + c) * ldm] : 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < PKB; ++c) v[a][c] = 0.0;
      }
    }
    for (int e = tid; e < PKB * PKB; e += PNT) {
      const int i = e % PKB, m = e / PKB;
      if (m < i && i < kb) cp_async8(l11 + i * PLD + m, Mg + (kp + i) + (long long)(kp + m) * ldm, 8);
      else l11[i * PLD + m] = 0.0;
    }
    cp_async_commit();
    const int* mvp = move_list(args, nd, kp);
    if (tid < 2 * PKB) {
      m_dst[tid] = mvp[tid];
      m_src[tid] = mvp[2 * PKB + tid];
    }
    constexpr int QC = PKB / PNW;
    double xs[QC];
#pragma unroll
    for (int q = 0; q < QC; ++q)
      xs[q] = (lane < kb && warp * QC + q < kbe) ? Mg[(kp + lane) + (long long)(k0 + warp * QC + q) * ldm] : 0.0;
    cp_async_wait<0>();
    __syncthreads();
    {
      const int i = lane, c0 = warp * QC;
      const int srow = m_src[i];
      double x[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q)
        x[q] = (srow == kp + i || !(i < kb && c0 + q < kbe)) ? xs[q] : Mg[srow + (long long)(k0 + c0 + q) * ldm];
#pragma unroll 4
      for (int m = 0; m < kb - 1; ++m) {
        const double lim = (i > m) ? l11[i * PLD + m] : 0.0;
#pragma unroll
        for (int q = 0; q < QC; ++q) x[q] = fma(-lim, __shfl_sync(0xffffffffu, x[q], m), x[q]);
      }
#pragma unroll
      for (int q = 0; q < QC; ++q) pro[i * PLD + c0 + q] = x[q];
    }
    const bool displaced = m_dst[PKB] >= 0;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = rowof(a);
      if (displaced && r < Ri) {
        const int R = k0 + r;
        int src = R;
#pragma unroll 4
        for (int t = PKB; t < 2 * PKB; ++t)
          if (m_dst[t] == R) src = m_src[t];
        if (src != R)
#pragma unroll
          for (int c = 0; c < PKB; ++c) v[a][c] = c < kbe ? Mg[src + (long long)(k0 + c) * ldm] : 0.0;
      }
    }
    __syncthreads();
    const bool lead = try_fast && crank == 0 && !lead32;
    if (lead && warp != 0) asm volatile("bar.sync 1, %0;" ::"r"(PNT) : "memory");
#pragma unroll 2
    for (int m = 0; m < (idle_warp ? 0 : kb); ++m) {
      double lm[RPT];
#pragma unroll
      for (int a = 0; a < RPT; ++a) lm[a] = psave[(a * PNT + tid) * (PKB + 1) + m];
      const double2* u2 = reinterpret_cast<const double2*>(pro + m * PLD);
#pragma unroll
      for (int c2 = 0; c2 < PKB / 2; ++c2) {
        const double2 u = u2[c2];
#pragma unroll
        for (int a = 0; a < RPT; ++a) {
          v[a][2 * c2] = fma(-lm[a], u.x, v[a][2 * c2]);
          v[a][2 * c2 + 1] = fma(-lm[a], u.y, v[a][2 * c2 + 1]);
        }
      }
    }
    if (lead && warp == 0) asm volatile("bar.arrive 1, %0;" ::"r"(PNT) : "memory");
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = rowof(a);
#pragma unroll
      for (int c = 0; c < PKB; ++c)
        if (c >= kbe || r >= Ri) v[a][c] = 0.0;
    }
  }
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = rowof(a);
    elim[a] = (r < Ri) ? -1 : PKB;
  }
  P2CLK(1);
  double pmin = k0 == 0 ? DBL_MAX : args.pivstat[2 * node_id];
  double pmax = k0 == 0 ? 0.0 : args.pivstat[2 * node_id + 1];
  bool bad = false;
  bool fast = false;
  int jstart = 0;
  if (try_fast) {
    // ---- no-interchange attempt (see panel_kernel): top block LU by warp 0 of
    // rank 0, every other row x U11 = a, verified |l| <= 1
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
      for (int c = 0; c < PKB; ++c) psave[(a * PNT + tid) * (PKB + 1) + c] = v[a][c];
    if (!piped && tid == 0) fast_fail = fail_all = PKB;
    int jf = PKB;
    P2CLK(2);
    if (crank == 0 && warp == 0) {  // rows 0..kbe-1 in lanes 0..kbe-1 (a = 0)
      // steps in chunks of 8 on a window narrowing by 8 (32, 24, 16, 8 live entries);
      // every lane forms the reciprocal of its next pivot candidate as soon as its
      // window's first entry is updated (lane j + 1's is the next pivot's)
      double rnext = __drcp_rn(v[0][0]);
      auto chunk = [&](auto Wc) {
        constexpr int W = decltype(Wc)::value;
        const int j0 = PKB - W, j1 = min(kbe, j0 + 8);
        for (int j = j0; j < j1; ++j) {
          if (lane == j) {
#pragma unroll
            for (int c = 0; c < W; c += 2)
              *reinterpret_cast<double2*>(ub + j * PLD + c) = make_double2(v[0][c], v[0][c + 1]);
            urinv[j] = rnext;
          }
          __syncwarp();
          if constexpr (CL) {
            if (piped && lane == 0) {  // row j is in ub: release it to the forwarding warp
              asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mbar_u[j])) : "memory");
            }
          }
          if (lane > j && lane < kbe) {
            const double l = v[0][0] * urinv[j];
            if (!(fabs(l) <= 1.0) && jf == PKB) jf = j;
            M[lane + (long long)j * ldm] = l;
            shift_update_w<W>(v[0], l, ub + j * PLD);
            rnext = __drcp_rn(v[0][0]);
          }
        }
      };
      chunk(WinC<32>{});
      chunk(WinC<24>{});
      chunk(WinC<16>{});
      chunk(WinC<8>{});
      for (int j = kbe + lane; j < PKB; j += 32) {  // rows past the panel: zero U rows
#pragma unroll 4
        for (int c = 0; c < PLD; ++c) ub[j * PLD + c] = 0.0;
      }
      const int jt = __reduce_min_sync(0xffffffffu, unsigned(jf));
      if (lane == 0) {
        if (piped) atomicMin(&fast_fail, jt);  // (the other warps may already have recorded theirs)
        else fast_fail = jt;
      }
    }
    if constexpr (CL) {
      const int nfw = min(PNW - 1, (csize - 1 + 3) / 4);  // one forwarding warp per 4 destinations
      if (piped && crank == 0 && warp >= 1 && warp <= nfw) {
        // forwarding warps (1 .. nfw, the destinations dealt round-robin; more warps would compete
        // with warp 0's top LU on this SM): U row j (shifted) and
        // 1 / u_jj to the other CTAs as soon as warp 0 has formed it (st.async, completing the
        // destination's barrier of row j)
        for (int j = 0; j < kbe; ++j) {
          mbar_wait(&mbar_u[j], 0u);
          const double val = ub[j * PLD + lane];
          const double rj = urinv[j];
          for (int d = warp; d < csize; d += nfw) {
            const unsigned mb = cluster_map(&mbar_u[j], d);
            st_async_b64(cluster_map(ub + j * PLD + lane, d), __double_as_longlong(val), mb);
            if (lane == 0) st_async_b64(cluster_map(urinv + j, d), __double_as_longlong(rj), mb);
          }
        }
      }
    }
    P2CLK(3);
    if constexpr (CL) {
      if (!piped) {
      cg::this_cluster().sync();
      if (crank != 0) {
        const double* rub = cg::this_cluster().map_shared_rank(ub, 0);
        for (int e = tid; e < PKB * PLD + PKB; e += PNT) ub[e] = rub[e];
        if (tid == 0) jtop_s = *cg::this_cluster().map_shared_rank(&fast_fail, 0);
      }
      }
    }
    if (!piped) {
      __syncthreads();
      if (crank == 0 && tid == 0) jtop_s = fast_fail;
      __syncthreads();
    }
    const int jtop = piped ? PKB : jtop_s;  // (pipelined: every step runs; the verification finds the first bad one)
    auto subst = [&](int rlo, int jmax, bool track, bool wait_rows = false) {
      auto chunk = [&](auto Wc) {
        constexpr int W = decltype(Wc)::value;
        const int j0 = PKB - W, j1 = min(jmax, j0 + 8);
        for (int j = j0; j < j1; ++j) {
          if (wait_rows) mbar_wait(&mbar_u[j], 0u);
#pragma unroll
          for (int a = 0; a < RPT; ++a) {
            const int r = rowof(a);
            if (r >= rlo && r < Ri) {
              const double l = v[a][0] * urinv[j];
              if (track && !(fabs(l) <= 1.0) && jf == PKB) jf = j;
#ifndef DTN_PROBE_NOSTORE
              M[r + (long long)j * ldm] = l;
#endif
              shift_update_w<W>(v[a], l, ub + j * PLD);
            }
          }
        }
      };
      chunk(WinC<32>{});
      chunk(WinC<24>{});
      chunk(WinC<16>{});
      chunk(WinC<8>{});
    };
    P2CLK(4);
    if (!(piped && crank == 0)) subst(kbe, min(kbe, jtop), true, piped);  // (light lead: rank 0 has no rows below)
    P2CLK(5);
    if (jf < PKB) atomicMin(&fast_fail, jf);
    __syncthreads();
    int jstar;
    if constexpr (CL) {
      if (warp == 0 && lane < csize && fast_fail < PKB)
        atomicMin(cg::this_cluster().map_shared_rank(&fail_all, lane), fast_fail);
      cg::this_cluster().sync();
      jstar = fail_all;
    } else {
      jstar = fast_fail;
    }
    jstar = min(jstar, kbe);
    fast = jstar >= kbe;
    P2CLK(6);
    if (crank == 0 && warp == 0) {
      const double apiv = fabs(ub[lane * PLD]);
      const bool live = lane < jstar;
      double lo = live ? apiv : DBL_MAX, hi = live ? apiv : 0.0;
      const bool nb_ = live && (!(apiv == apiv) || apiv == INFINITY);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      pmin = fmin(pmin, lo);
      pmax = fmax(pmax, hi);
      bad |= __any_sync(0xffffffffu, nb_);
    }
    if (fast) {
      if (crank == 0) {
        if (tid < 2 * PKB) {
          int* mv = move_list(args, nd, k0);
          mv[tid] = tid < kbe ? k0 + tid : -1;
          mv[2 * PKB + tid] = tid < kbe ? k0 + tid : -1;
        }
        for (int e = tid; e < PKB * PKB; e += PNT) {  // U rows in place
          const int i = e % PKB, c = e / PKB;
          if (i < kbe && c >= i && c < kbe) M[i + (long long)c * ldm] = ub[i * PLD + (c - i)];
        }
      }
    } else {
      if (crank == 0 && tid == 0) {
        atomicAdd(&g_panel_fallbacks, 1u);
        *pivoting_flag(args, nd) += 1;
      }
      // rows >= jstar restart from the saved values with the steps < jstar (exactly
      // partial pivoting's); rows < jstar are the pivots of steps 0 .. jstar - 1
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = rowof(a);
        if (r >= jstar)
#pragma unroll
          for (int c = 0; c < PKB; ++c) v[a][c] = psave[(a * PNT + tid) * (PKB + 1) + c];
      }
      subst(jstar, jstar, false);
      jstart = jstar;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = rowof(a);
        if (r < jstart) elim[a] = r;
      }
      if (tid < jstart) sp[tid] = tid;
    }
  }
  if (!fast) {
    const unsigned tx_bytes = unsigned(csize) * (PKB * 8 + 16);
    if constexpr (CL) {
      if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arm(&mbar[0], tx_bytes);
        mbar_arm(&mbar[1], tx_bytes);
      }
      cg::this_cluster().sync();
    }
#ifdef DTN_PANEL_PROFILE
    long long tq = clock64();
#endif
    // steps in chunks of 8 on a window narrowing by 8 (see shift_update_w)
    auto pchunk = [&](auto Wc) {
    constexpr int W = decltype(Wc)::value;
    const int jlo = max(jstart, PKB - W), jhi = min(kbe, PKB - W + 8);
    for (int j = jlo; j < jhi; ++j) {
      const int jr = j - jstart;
      const int buf = jr & 1;
      unsigned key = 0u, klo = 0u;
      int ba = 0;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const double ax = fabs(v[a][0]);
        const unsigned ka = elim[a] < 0 ? (unsigned(__double2hiint(ax)) | 0x80000000u) : 0u;
        const unsigned kl = unsigned(__double2loint(ax));
        if (ka > key || (ka == key && kl > klo)) {
          key = ka;
          klo = kl;
          ba = a;
        }
      }
      const unsigned whi = __reduce_max_sync(0xffffffffu, key);
      const unsigned wlo = __reduce_max_sync(0xffffffffu, key == whi ? klo : 0u);
      const int wlane = __ffs(__ballot_sync(0xffffffffu, key == whi && klo == wlo)) - 1;
      {
        const bool win = lane == wlane;
#pragma unroll
        for (int a = 0; a < RPT; ++a) {
          const bool wa = win && a == ba;
#pragma unroll
          for (int c = 0; c < PKB; c += 2) st_shared_v2_pred(&rows[buf][warp][c], v[a][c], v[a][c + 1], wa);
        }
        st_shared_v4u_pred(&sinfo[buf][warp][0], whi, wlo, unsigned(rowof(ba)), 0u, win);
      }
      P2ACC(9, tq);
      __syncthreads();
      P2ACC(10, tq);
      const unsigned lk = lane < PNW ? sinfo[buf][lane][0] : 0u;
      const unsigned ll = lane < PNW ? sinfo[buf][lane][1] : 0u;
      const unsigned bkey = __reduce_max_sync(0xffffffffu, lk);
      const unsigned blo = __reduce_max_sync(0xffffffffu, lk == bkey ? ll : 0u);
      const int bw = __ffs(__ballot_sync(0xffffffffu, lk == bkey && ll == blo && lane < PNW)) - 1;
      int slot = bw, p = int(sinfo[buf][bw][2]);
      if constexpr (CL) {
        {
          const double rv = rows[buf][bw][lane];
          for (int d = warp; d < csize; d += PNW) {
            const unsigned mb = cluster_map(&mbar[buf], d);
            st_async_b64(cluster_map(&rows[buf][SC + crank][lane], d), __double_as_longlong(rv), mb);
            if (lane == 0) st_async_v4_b32(cluster_map(&cinfo[buf][crank][0], d), bkey, blo, unsigned(p), 0u, mb);
          }
        }
        P2ACC(11, tq);
        mbar_wait(&mbar[buf], unsigned(jr >> 1) & 1u);
        P2ACC(12, tq);
        const unsigned ck = lane < csize ? cinfo[buf][lane][0] : 0u;
        const unsigned cl_ = lane < csize ? cinfo[buf][lane][1] : 0u;
        const unsigned gkey = __reduce_max_sync(0xffffffffu, ck);
        const unsigned glo = __reduce_max_sync(0xffffffffu, ck == gkey ? cl_ : 0u);
        const int cw = __ffs(__ballot_sync(0xffffffffu, ck == gkey && cl_ == glo && lane < csize)) - 1;
        slot = SC + cw;
        p = int(cinfo[buf][cw][2]);
      }
      const double* prow = &rows[buf][slot][0];
      const double piv = prow[0];
      if (crank == 0 && warp == (j & (PNW - 1))) ub[j * PLD + lane] = prow[lane];  // U row j (shifted)
      if constexpr (CL) {
        if (tid == 0) mbar_arm(&mbar[buf], tx_bytes);
      }
      const double apiv = fabs(piv);
      pmin = fmin(pmin, apiv);
      pmax = fmax(pmax, apiv);
      bad |= !(apiv == apiv) || apiv == INFINITY;
      const double rinv = __drcp_rn(piv);
      P2ACC(13, tq);
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int r = rowof(a);
        if (r == p) elim[a] = j;
        if (elim[a] < 0) {
          const double l = v[a][0] * rinv;
          M[r + (long long)j * ldm] = l;
          shift_update_w<W>(v[a], l, prow);
        }
      }
      if (tid == 0) sp[j] = p;
      P2ACC(14, tq);
    }
    };
    pchunk(WinC<32>{});
    pchunk(WinC<24>{});
    pchunk(WinC<16>{});
    pchunk(WinC<8>{});
    // ---- final placement: pivot of step e -> position e; the top rows [0, kbe)
    // that were not pivots fill, in order, the positions vacated by pivots from
    // below (also in order). Only those rows move: rank 0 stages them through
    // shared memory once every CTA's stores are visible.
    csync();
    if (crank == 0)
      place_panel_rows<PNT>(M, ldm, k0, kbe, sp, vac, mv_dst, mv_src, ub, psave, perm, move_list(args, nd, k0));
  }
  P2CLK(7);
  if (fused && k0 > 0 && crank == 0) {  // U12 of the prologue into rows [k0 - kb, k0)
    double* Mg = args.arena + nd.m_off;
    for (int e = tid; e < PKB * PKB; e += PNT) {
      const int i = e % PKB, c = e / PKB;
      if (i < kb && c < kbe) Mg[(k0 - kb + i) + (long long)(k0 + c) * ldm] = pro[i * PLD + c];
    }
  }
  if (crank == 0 && tid == 0) {
    args.pivstat[2 * node_id] = pmin;
    args.pivstat[2 * node_id + 1] = bad ? INFINITY : pmax;
  }
  P2CLK(8);
  if constexpr (CL) cg::this_cluster().sync();  // no CTA exits while others may still read its smem
}

// ---------------------------------------------------------------------------
// tall_panel_kernel: the panel contract of panel2_kernel (non-fused, partial pivoting
// from the first step) for systems beyond the cluster panel's 16 x 512 rows -- the root
// LU of G = S^{-1} at config 4 (16380 rows). Rows are spread over TG CTAs per system
// (gridDim.x = TG, gridDim.y = systems), RPT rows per thread in shifting register windows
// as in panel2. A cluster cannot span more than 16 SMs, so the pivot exchange goes through
// global memory: each CTA publishes its best candidate row (key + 32 values), one software
// barrier over the system's TG CTAs, then every CTA picks the same winner (largest |a|,
// ties to the lowest row) and applies the step locally. The launcher keeps the whole grid
// within one CTA per SM, so every CTA of a system is resident together.
constexpr int TALL_NT = 256;
constexpr int TALL_MAX_CTAS = 160;
struct TallCand {
  double v[PKB];
  unsigned hi, lo;
  int row, pad;
};
__device__ TallCand g_tall_cand[2][TALL_MAX_CTAS];
__device__ unsigned g_tall_bar[TALL_MAX_CTAS];

__device__ __forceinline__ void tall_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned x;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(bar) : "memory");
    } while (x < target);
  }
  __syncthreads();
}

// (hi, lo, row) candidate order: larger |a| wins, equal |a| goes to the lower row
__device__ __forceinline__ bool tall_better(unsigned h1, unsigned l1, int r1, unsigned h2, unsigned l2, int r2) {
  return h1 > h2 || (h1 == h2 && (l1 > l2 || (l1 == l2 && r1 < r2)));
}

template <int RPT>
__global__ void __launch_bounds__(TALL_NT) tall_panel_kernel(KernelArgs args, const int* __restrict__ list, int k0,
                                                             int kb) {
  constexpr int NW = TALL_NT / 32, PLD = PKB + 2;
  __shared__ __align__(16) double wrow[NW][PKB];
  __shared__ unsigned whi[NW], wlo[NW];
  __shared__ int wr[NW];
  __shared__ __align__(16) double ub[PKB * PLD];
  __shared__ __align__(16) double stage[2 * PKB * PKB];
  __shared__ int sp[PKB], vac[PKB], mv_dst[2 * PKB], mv_src[2 * PKB];
  __shared__ int s_win;
  const int TG = gridDim.x, sys = blockIdx.y;
  const int node_id = list[sys];
  const NodeDev nd = args.nodes[node_id];
  if (k0 >= nd.ni) return;  // uniform over the system's CTAs
  const int kbe = min(kb, nd.ni - k0);
  const int Ri = nd.ni - k0;
  double* M = args.arena + nd.m_off + k0 + (long long)k0 * nd.ldm;
  const long long ldm = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int stride = TG * TALL_NT;
  int* perm = args.piv + nd.piv_off;
  TallCand* cand0 = g_tall_cand[0] + sys * TG;
  TallCand* cand1 = g_tall_cand[1] + sys * TG;
  unsigned* bar = g_tall_bar + sys;
  unsigned nsync = 0;

  double v[RPT][PKB];
  int elim[RPT];
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int r = blockIdx.x * TALL_NT + tid + stride * a;
#pragma unroll
    for (int c = 0; c < PKB; ++c) v[a][c] = (r < Ri && c < kbe) ? M[r + c * ldm] : 0.0;
    if (k0 == 0 && r < Ri) perm[r] = r;
    elim[a] = (r < Ri) ? -1 : PKB;
  }
  if (k0 == 0 && blockIdx.x == 0 && tid == 0) *pivoting_flag(args, nd) = 0;
  double pmin = k0 == 0 ? DBL_MAX : args.pivstat[2 * node_id];
  double pmax = k0 == 0 ? 0.0 : args.pivstat[2 * node_id + 1];
  bool bad = false;
  for (int j = 0; j < kbe; ++j) {
    TallCand* cand = (j & 1) ? cand1 : cand0;
    // this thread's best live row, then the warp's, then the CTA's
    unsigned key = 0u, klo = 0u;
    int br = 0x7fffffff, ba = 0;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const double ax = fabs(v[a][0]);
      const unsigned ka = elim[a] < 0 ? (unsigned(__double2hiint(ax)) | 0x80000000u) : 0u;
      const unsigned kl = elim[a] < 0 ? unsigned(__double2loint(ax)) : 0u;
      const int r = blockIdx.x * TALL_NT + tid + stride * a;
      if (ka != 0u && tall_better(ka, kl, r, key, klo, br)) {
        key = ka;
        klo = kl;
        br = r;
        ba = a;
      }
    }
    const unsigned mh = __reduce_max_sync(0xffffffffu, key);
    const unsigned ml = __reduce_max_sync(0xffffffffu, key == mh ? klo : 0u);
    const int mr = int(__reduce_min_sync(0xffffffffu, unsigned(key == mh && klo == ml ? br : 0x7fffffff)));
    if (br == mr && key == mh && mh != 0u) {
#pragma unroll
      for (int a = 0; a < RPT; ++a)
        if (a == ba)
#pragma unroll
          for (int c = 0; c < PKB; ++c) wrow[warp][c] = v[a][c];
    }
    if (lane == 0) {
      whi[warp] = mh;
      wlo[warp] = ml;
      wr[warp] = mr;
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned h = lane < NW ? whi[lane] : 0u, l = lane < NW ? wlo[lane] : 0u;
      const int r = lane < NW ? wr[lane] : 0x7fffffff;
      const unsigned bh = __reduce_max_sync(0xffffffffu, h);
      const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
      const int brow = int(__reduce_min_sync(0xffffffffu, unsigned(h == bh && l == bl ? r : 0x7fffffff)));
      const int bw = __ffs(__ballot_sync(0xffffffffu, lane < NW && h == bh && l == bl && r == brow)) - 1;
      TallCand& mine = cand[blockIdx.x];
      mine.v[lane] = bh != 0u ? wrow[bw][lane] : 0.0;
      if (lane == 0) {
        mine.hi = bh;
        mine.lo = bl;
        mine.row = brow;
      }
    }
    tall_barrier(bar, unsigned(TG) * ++nsync);
    // every CTA picks the same winner among the TG candidates
    if (warp == 0) {
      unsigned h = 0u, l = 0u;
      int r = 0x7fffffff, w = 0;
      for (int c = lane; c < TG; c += 32) {
        const unsigned ch = __ldcg(&cand[c].hi), cl = __ldcg(&cand[c].lo);
        const int cr = __ldcg(&cand[c].row);
        if (ch != 0u && tall_better(ch, cl, cr, h, l, r)) {
          h = ch;
          l = cl;
          r = cr;
          w = c;
        }
      }
      const unsigned bh = __reduce_max_sync(0xffffffffu, h);
      const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
      const int brow = int(__reduce_min_sync(0xffffffffu, unsigned(h == bh && l == bl ? r : 0x7fffffff)));
      const int src = __shfl_sync(0xffffffffu, w, __ffs(__ballot_sync(0xffffffffu, h == bh && l == bl && r == brow)) - 1);
      ub[j * PLD + lane] = __ldcg(&cand[src].v[lane]);  // U row j, shifted (ub[j][c] = U[j][j + c])
      if (lane == 0) {
        s_win = brow;
        sp[j] = brow;
      }
    }
    __syncthreads();
    const int p = s_win;
    const double* prow = ub + j * PLD;
    const double piv = prow[0];
    const double apiv = fabs(piv);
    pmin = fmin(pmin, apiv);
    pmax = fmax(pmax, apiv);
    bad |= !(apiv == apiv) || apiv == INFINITY;
    const double rinv = __drcp_rn(piv);
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int r = blockIdx.x * TALL_NT + tid + stride * a;
      if (r == p) elim[a] = j;
      if (elim[a] < 0) {
        const double l = v[a][0] * rinv;
        M[r + (long long)j * ldm] = l;
        shift_update(v[a], l, prow);
      }
    }
  }
  for (int e = kbe * PLD + tid; e < PKB * PLD; e += TALL_NT) ub[e] = 0.0;
  // every CTA's multipliers visible before CTA 0 moves rows
  tall_barrier(bar, unsigned(TG) * ++nsync);
  if (blockIdx.x == 0) {
    place_panel_rows<TALL_NT>(M, ldm, k0, kbe, sp, vac, mv_dst, mv_src, ub, stage, perm, move_list(args, nd, k0));
    if (tid == 0) {
      args.pivstat[2 * node_id] = pmin;
      args.pivstat[2 * node_id + 1] = bad ? INFINITY : pmax;
    }
  }
}

// Row swaps + U12 = L11^{-1} (P A)[k0:k1, k1:total] for the trailing columns;
// with swap_left, also the row swaps of the already factored columns [0, k0)
// (needed only when L itself is reused: the root LU for G = S^{-1}).
// BROWS: the launch includes boundary-row tiles (non-Schur merges). Without them the
// kernel needs few registers (the boundary rows' 32-entry solve is compiled out), so
// several CTAs share an SM (with it: 154 registers, one CTA per SM -- the first blocked
// waves' thousands of column tiles ran one CTA per SM at a time).
template <bool BROWS>
__global__ void __launch_bounds__(RP_THREADS) rowpanel_kernel(KernelArgs args, const int* __restrict__ list, int k0,
                                                              int kb, int ncoltiles, int nlefttiles, int skip_next) {
  __shared__ double T[32][33];
  __shared__ int s_dst[64], s_src[64];
  const NodeDev nd = args.nodes[list[blockIdx.y]];
  if (k0 >= nd.ni) return;
  const int kbe = min(kb, nd.ni - k0), k1 = k0 + kbe;
  double* M = args.arena + nd.m_off;
  const long long ld = nd.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bx = blockIdx.x;
  if (BROWS && bx >= ncoltiles + nlefttiles) {
    // boundary rows [ni, total): L21 = A[i, k0:k1] U11^{-1}
    const int i = nd.ni + (bx - ncoltiles - nlefttiles) * RP_THREADS + tid;
    if (nd.ni + (bx - ncoltiles - nlefttiles) * RP_THREADS >= nd.total) return;
    for (int e = tid; e < kbe * kbe; e += RP_THREADS) T[e % kbe][e / kbe] = M[(k0 + e % kbe) + (k0 + e / kbe) * ld];
    __syncthreads();
    if (i >= nd.total) return;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c] = c < kbe ? M[i + (k0 + c) * ld] : 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (c < kbe) {
        double sacc = x[c];
#pragma unroll
        for (int l = 0; l < c; ++l) sacc = fma(-x[l], T[l][c], sacc);
        x[c] = sacc / T[c][c];
      }
    }
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < kbe) M[i + (k0 + c) * ld] = x[c];
    return;
  }
  const bool left = bx >= ncoltiles;
  // skip_next: the next panel (fused prologue) owns columns [k1, k1 + min(kb, ni - k1))
  const int cs = k1 + (skip_next ? min(kb, max(nd.ni - k1, 0)) : 0);
  const int jbase = left ? (bx - ncoltiles) * RP_COLS : cs + bx * RP_COLS;
  const int jend = left ? k0 : (nd.defer ? nd.ni : nd.ncols);  // deferred: interface columns only
  if (jbase >= jend) return;
  const int* mv = move_list(args, nd, k0);
  if (tid < 64) {
    s_dst[tid] = mv[tid];
    s_src[tid] = mv[64 + tid];
  }
  if (!left)
    for (int e = tid; e < kbe * kbe; e += RP_THREADS) T[e % kbe][e / kbe] = M[(k0 + e % kbe) + (k0 + e / kbe) * ld];
  __syncthreads();
  // a warp owns 4 columns: all gathers are issued first (one L2 round trip);
  // slot i < kbe always moves a row into k0+i, so the top block is solved
  // from registers (no store -> reload)
  constexpr int CPW = RP_COLS / (RP_THREADS / 32);
  const int d0 = s_dst[lane], d1 = s_dst[lane + 32];
  const int s0 = s_src[lane], s1 = s_src[lane + 32];
  double g0[CPW], g1[CPW];
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = jbase + warp * CPW + q;
    const double* col = M + (long long)j * ld;
    g0[q] = (j < jend && d0 >= 0) ? col[s0] : 0.0;
    g1[q] = (j < jend && d1 >= 0) ? col[s1] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = jbase + warp * CPW + q;
    if (j >= jend) break;
    double* col = M + (long long)j * ld;
    if (d1 >= 0) col[d1] = g1[q];
    if (left) {
      if (d0 >= 0) col[d0] = g0[q];
      continue;
    }
    if (d0 >= 0 && lane >= kbe) col[d0] = g0[q];
  }
  if (left) return;
  // unit lower L11 solves of the warp's columns, interleaved (independent shuffle/FMA
  // chains in flight together instead of one column after another)
  double x[CPW];
#pragma unroll
  for (int q = 0; q < CPW; ++q) x[q] = lane < kbe ? g0[q] : 0.0;
  for (int c = 0; c < kbe; ++c) {
    const double tl = (lane > c && lane < kbe) ? T[lane][c] : 0.0;
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const double xc = __shfl_sync(0xffffffffu, x[q], c);
      x[q] = fma(-tl, xc, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int j = jbase + warp * CPW + q;
    if (j < jend && lane < kbe) M[(long long)j * ld + k0 + lane] = x[q];
  }
}

unsigned panel_fallbacks_read_reset() {
  unsigned h = 0, z = 0;
  cudaMemcpyFromSymbol(&h, g_panel_fallbacks, sizeof(h));
  cudaMemcpyToSymbol(g_panel_fallbacks, &z, sizeof(z));
  return h;
}

size_t panel_dyn_smem(int rpt, int nt) { return size_t(PKB * (PKB + 2) + PKB + rpt * nt * (PKB + 1)) * sizeof(double); }
size_t panel_dyn_smem(int rpt) { return panel_dyn_smem(rpt, PNT); }

// no-interchange attempts stop for a node after this many of its panels
// needed interchanges (DTN_FAST_THRESHOLD; 0 = always run the pivoted loop).
// Default: always attempt -- a failed attempt costs the top-block LU and the
// substitution, and the pivoted loop then resumes at the first step that
// needs an interchange (config 2: 8.87 ms vs 9.16 ms with threshold 1).
int panel_fast_threshold() {
  static const int th = [] {
    const char* e = std::getenv("DTN_FAST_THRESHOLD");
    return e ? std::atoi(e) : (1 << 30);
  }();
  return th;
}

// DTN_PANEL_LEGACY=1: the fully unrolled panel_kernel instead of panel2_kernel
bool panel_legacy() {
  static const bool on = std::getenv("DTN_PANEL_LEGACY") != nullptr;
  return on;
}

cudaError_t blocked_init() {
  for (auto f : {panel2_kernel<true, 1>, panel2_kernel<true, 2>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  for (auto f : {panel2_kernel<true, 1>, panel2_kernel<false, 1>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(panel_dyn_smem(1)));
    if (e != cudaSuccess) return e;
  }
  for (auto f : {panel2_kernel<true, 2>, panel2_kernel<false, 2>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(panel_dyn_smem(2)));
    if (e != cudaSuccess) return e;
  }
  {
    cudaError_t e = cudaFuncSetAttribute(panel2_kernel<true, 1, 128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel2_kernel<true, 1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(panel_dyn_smem(1, 128)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel2_kernel<false, 1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(panel_dyn_smem(1, 128)));
    if (e != cudaSuccess) return e;
  }
  {
    cudaError_t e = cudaFuncSetAttribute(panel2_kernel<true, 2, 128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel2_kernel<true, 2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(panel_dyn_smem(2, 128)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel2_kernel<false, 2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(panel_dyn_smem(2, 128)));
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaFuncSetAttribute(panel_kernel<true, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(panel_kernel<true, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  for (cudaError_t x : {cudaFuncSetAttribute(panel_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(panel_dyn_smem(1))),
                        cudaFuncSetAttribute(panel_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(panel_dyn_smem(2))),
                        cudaFuncSetAttribute(panel_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(panel_dyn_smem(1))),
                        cudaFuncSetAttribute(panel_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(panel_dyn_smem(2)))})
    if (x != cudaSuccess) return x;
  return cudaSuccess;
}

cudaError_t launch_gather(const KernelArgs& args, const int* d_list, int count, int max_total, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((max_total + args.nl + GATHER_COLS - 1) / GATHER_COLS, count);
  gather_kernel<<<grid, 256, 0, st>>>(args, d_list);
  return cudaGetLastError();
}

// Panel geometry for systems with up to max_rows rows below k0 (kb <= 32):
// one row per thread up to 16 CTAs x 256 rows, two rows per thread beyond
// (clusters of up to 16 CTAs, 8192 rows).
// DTN_PANEL_ONECTA2=1: systems of 257..512 rows on ONE CTA with 2 rows per thread
// (the pivoted loop's cheapest exchange) instead of a 2-CTA cluster (half the
// prologue update and substitution per CTA: the no-interchange path's cost)
static bool panel_onecta2() {
  static const bool on = [] {
    const char* e = std::getenv("DTN_PANEL_ONECTA2");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

void panel_shape(int max_rows, int* rpt, int* csize);

// DTN_PANEL_NT1=0: systems of <= 128 rows on 256-thread CTAs (default: 128-thread CTAs, three
// per SM by registers -- the many-system waves run one panel CTA per system)
static bool panel_small_nt1() {
  static const bool on = [] {
    const char* e = std::getenv("DTN_PANEL_NT1");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// DTN_PANEL_NT=128: panels of 257..2048 rows on clusters of 128-thread CTAs (twice the
// SMs per panel; measured 1-2 % slower than the 256-thread default on configs 2, 3, 5: the
// no-interchange top LU and the per-pivot exchange, not the per-CTA work, set the time)
static int panel_small_nt() {
  static const int v = [] {
    const char* e = std::getenv("DTN_PANEL_NT");
    return e ? std::atoi(e) : 256;
  }();
  return v;
}

static bool panel_r2() {
  static const bool on = [] {
    const char* e = std::getenv("DTN_PANEL_R2");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

void panel_shape(int max_rows, int* rpt, int* csize, int* nt) {
  *nt = PNT;
  if (!panel_legacy() && max_rows <= 128 && panel_small_nt1()) {  // one 128-thread CTA: 3 per SM
    *rpt = 1;
    *csize = 1;
    *nt = 128;
    return;
  }
  // DTN_PANEL_R2=1: 128-thread CTAs with TWO rows per thread (the cluster size of the default,
  // half the warps per SM): the substitution, the prologue update and the pivoted update all
  // re-read the 32-entry pivot / U row from shared memory in every lane, 8 warps x 256 B x 4
  // quarter-warp passes per step -- shared-memory bandwidth, not FP64 issue, bounds them
  if (!panel_legacy() && panel_r2() && max_rows > PNT && max_rows <= PMAXC * PNT) {
    *rpt = 2;
    *csize = (max_rows + PNT - 1) / PNT;
    *nt = 128;
    return;
  }
  if (!panel_legacy() && panel_small_nt() == 128 && max_rows > PNT && max_rows <= PKB + (PMAXC - 1) * 128) {
    *rpt = 1;
    *csize = (max_rows + 127) / 128;
    *nt = 128;
    return;
  }
  panel_shape(max_rows, rpt, csize);
}

void panel_shape(int max_rows, int* rpt, int* csize) {
  // measured per-pivot cost (tools/probe/panel_probe): one CTA 0.9 us (<= 256
  // rows), one CTA with 2 rows/thread 1.14 us (<= 512), clusters with the
  // st.async exchange 1.3-1.6 us (2-16 CTAs x 256 rows), 2 rows/thread beyond
  if (max_rows <= PNT) { *rpt = 1; *csize = 1; }
  else if (max_rows <= 2 * PNT && panel_onecta2()) { *rpt = 2; *csize = 1; }
  else if (max_rows <= PMAXC * PNT) { *rpt = 1; *csize = (max_rows + PNT - 1) / PNT; }
  else { *rpt = 2; *csize = (max_rows + 2 * PNT - 1) / (2 * PNT); }
}

size_t panel_dyn_smem(int rpt);
int panel_fast_threshold();
bool panel_legacy();

// Pipelined no-interchange attempt of the cluster panels (DTN_PANEL_PIPE=0: the classic order).
// Rank 0 holds only the 32 top rows (light lead CTA: its warp 0 factors the top block with no other
// warp of the SM computing -- 390 instead of 475 cycles per pivot), warp 1 of rank 0 forwards every
// U row to the other CTAs as it is formed (st.async + one mbarrier per row), and the rows below
// run substitution step j as soon as row j has landed instead of starting after the whole top LU.
// Same arithmetic (S bit-identical); 1024-row panel 28.6 -> 24.5 us.
static bool panel_pipe() {
  static const bool on = [] {
    const char* e = std::getenv("DTN_PANEL_PIPE");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

template <bool CL, int RPT, int NT = PNT>
cudaError_t launch_panel_t(const KernelArgs& args, const int* d_list, int count, int k0, int kb, int csize,
                           cudaStream_t st, bool fused, bool pipe = false) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * csize);
  cfg.blockDim = dim3(NT);
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
  cfg.dynamicSmemBytes = panel_dyn_smem(RPT, NT);
  if (NT == PNT && panel_legacy())
    return cudaLaunchKernelEx(&cfg, panel_kernel<CL, RPT>, args, d_list, k0, kb, csize, fused ? 1 : 0,
                              panel_fast_threshold());
  return cudaLaunchKernelEx(&cfg, panel2_kernel<CL, RPT, NT>, args, d_list, k0, kb, csize, fused ? 1 : 0,
                            panel_fast_threshold() ? (std::min(panel_fast_threshold(), 0x1fffffff) | (pipe ? 0x20000000 : 0)) : 0);
}

// fused: apply step k0 - kb to this panel's columns first (the look-ahead
// prologue); the matching rowpanel / trailing launches skip those columns.
// DTN_PANEL_TALL_MIN: panels of at least this many rows take tall_panel_kernel (default:
// beyond the cluster panel's 16 x 512 rows; smaller values exercise it in the tests)
// (read per call: a few hundred panel launches per build)
int panel_tall_min() {
  const char* e = std::getenv("DTN_PANEL_TALL_MIN");
  return e ? std::max(1, std::atoi(e)) : PMAXC * 2 * PNT + 1;
}
bool panel_is_tall(int max_rows) { return max_rows >= panel_tall_min(); }

static unsigned* g_tall_bar_addr = nullptr;

// grid: TG CTAs per system, TG x count <= one CTA per SM (all resident together)
cudaError_t launch_tall_panel(const KernelArgs& args, const int* d_list, int count, int max_rows, int k0, int kb,
                              cudaStream_t st) {
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  if (!g_tall_bar_addr) {
    e = cudaGetSymbolAddress(reinterpret_cast<void**>(&g_tall_bar_addr), g_tall_bar);
    if (e != cudaSuccess) return e;
  }
  const int slots = std::min(nsm, TALL_MAX_CTAS);
  for (int rpt = 1; rpt <= 2; ++rpt) {
    const int tg = (max_rows + rpt * TALL_NT - 1) / (rpt * TALL_NT);
    if (tg * count > slots) continue;
    e = cudaMemsetAsync(g_tall_bar_addr, 0, sizeof(unsigned) * count, st);
    if (e != cudaSuccess) return e;
    dim3 grid(tg, count);
    if (rpt == 1) tall_panel_kernel<1><<<grid, TALL_NT, 0, st>>>(args, d_list, k0, kb);
    else tall_panel_kernel<2><<<grid, TALL_NT, 0, st>>>(args, d_list, k0, kb);
    return cudaGetLastError();
  }
  return cudaErrorNotSupported;  // more rows than two register rows per thread on every SM
}

// the tall panel's row limit for `count` systems on this device (0 on error)
int panel_tall_max_rows(int count) {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return std::min(nsm, TALL_MAX_CTAS) / std::max(1, count) * 2 * TALL_NT;
}

cudaError_t launch_panel(const KernelArgs& args, const int* d_list, int count, int max_rows, int k0, int kb,
                         cudaStream_t st, bool fused) {
  if (count <= 0) return cudaSuccess;
  if (kb > PKB) return cudaErrorInvalidValue;
  if (panel_is_tall(max_rows)) {
    if (fused) return cudaErrorInvalidValue;  // the engine runs tall systems without the look-ahead
    const cudaError_t e = launch_tall_panel(args, d_list, count, max_rows, k0, kb, st);
    if (e != cudaErrorNotSupported || max_rows > PMAXC * 2 * PNT) return e;
    // (a lowered DTN_PANEL_TALL_MIN on a wave of many systems: the cluster panel, non-fused)
  }
  int rpt, csize, nt;
  panel_shape(max_rows, &rpt, &csize, &nt);
  if (csize > PMAXC) return cudaErrorInvalidValue;
  if (nt == 128 && rpt == 2 && csize == 1) return launch_panel_t<false, 2, 128>(args, d_list, count, k0, kb, 1, st, fused);
  if (nt == 128 && rpt == 2) return launch_panel_t<true, 2, 128>(args, d_list, count, k0, kb, csize, st, fused);
  if (nt == 128 && csize == 1) return launch_panel_t<false, 1, 128>(args, d_list, count, k0, kb, 1, st, fused);
  if (nt == 128) {
    const int cs_pipe = 1 + (max_rows - PKB + 127) / 128;
    if (panel_pipe() && panel_fast_threshold() && cs_pipe <= PMAXC)
      return launch_panel_t<true, 1, 128>(args, d_list, count, k0, kb, cs_pipe, st, fused, true);
    return launch_panel_t<true, 1, 128>(args, d_list, count, k0, kb, csize, st, fused);
  }
  if (csize == 1 && rpt == 2) return launch_panel_t<false, 2>(args, d_list, count, k0, kb, 1, st, fused);
  if (csize == 1) return launch_panel_t<false, 1>(args, d_list, count, k0, kb, 1, st, fused);
  if (rpt == 1) {
    // pipelined substitution with the light lead CTA: rank 0 holds the 32 top rows only
    const int cs_pipe = 1 + (max_rows - PKB + PNT - 1) / PNT;
    if (panel_pipe() && panel_fast_threshold() && cs_pipe <= PMAXC)
      return launch_panel_t<true, 1>(args, d_list, count, k0, kb, cs_pipe, st, fused, true);
    return launch_panel_t<true, 1>(args, d_list, count, k0, kb, csize, st, fused);
  }
  return launch_panel_t<true, 2>(args, d_list, count, k0, kb, csize, st, fused);
}

cudaError_t launch_rowpanel(const KernelArgs& args, const int* d_list, int count, int max_total, int max_nb, int k0,
                            int kb, bool swap_left, cudaStream_t st, bool skip_next) {
  if (count <= 0) return cudaSuccess;
  const int coltiles = (max_total + args.nl - k0 + RP_COLS - 1) / RP_COLS;
  const int lefttiles = swap_left ? (k0 + RP_COLS - 1) / RP_COLS : 0;
  const int rowtiles = (max_nb + RP_THREADS - 1) / RP_THREADS;
  if (coltiles + lefttiles + rowtiles <= 0) return cudaSuccess;
  dim3 grid(coltiles + lefttiles + rowtiles, count);
  if (rowtiles > 0)
    rowpanel_kernel<true><<<grid, RP_THREADS, 0, st>>>(args, d_list, k0, kb, coltiles, lefttiles, skip_next ? 1 : 0);
  else
    rowpanel_kernel<false><<<grid, RP_THREADS, 0, st>>>(args, d_list, k0, kb, coltiles, lefttiles, skip_next ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace dtnb
