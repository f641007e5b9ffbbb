// Fused one-CTA elimination for small systems (total <= 160 unknowns):
//  * micro boxes below a reference leaf: assemble A over the box's nodes
//    ordered [interior row-major; boundary CCW] from the stencil and
//    eliminate the interior — leaf_schur, dense_nd.cpp:37-103;
//  * small pairwise merges: assemble the merge system from the two child
//    Schur complements plus the cross-interface couplings and eliminate the
//    interface — merge_two, dense_nd.cpp:135-181.
// The system lives in registers, distributed over a TR x TC thread grid
// (thread (tr,tc) owns rows tr+TR*a and columns tc+TC*b). Elimination is
// Gaussian elimination with partial pivoting restricted to the eliminated
// rows (PartialPivLU of M_ii, dense_nd.cpp:174) done without physical row
// swaps: pivot rows are flagged instead of moved, so the boundary rows end up
// holding S = M_bb - M_bi M_ii^{-1} M_ib in place. Two __syncthreads per pivot.
#include <cfloat>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace dtnb {

__device__ __forceinline__ void st_shared_f64_pred(double* p, double v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}" ::"r"(smem_u32(p)), "d"(v),
               "r"(int(pred))
               : "memory");
}
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ unsigned g_small_fallbacks;  // small systems whose no-interchange attempt failed (diagnostic)
unsigned small_fallbacks_read_reset() {
  unsigned h = 0, z = 0;
  cudaMemcpyFromSymbol(&h, g_small_fallbacks, sizeof(h));
  cudaMemcpyToSymbol(g_small_fallbacks, &z, sizeof(z));
  return h;
}

template <int TR, int TC, int RPT, int CPT, bool MICRO>
__global__ void __launch_bounds__(TR * TC) small_elim_kernel(KernelArgs args, const int* __restrict__ list) {
  constexpr int MAXT = (TR * RPT > TC * CPT) ? TR * RPT : TC * CPT;
  static_assert(TR <= 32 && (32 % TR) == 0, "column-owner group must sit inside one warp");
  __shared__ PosDev spos[MAXT];
  __shared__ double sst[MICRO ? 5 : 1][MICRO ? MAXT : 1];
  __shared__ double colk[2][MAXT];
  __shared__ double rowp[MAXT];
  __shared__ int s_piv;
  __shared__ double s_rinv;

  const int node_id = list[blockIdx.x];
  const NodeDev nd = args.nodes[node_id];
  const int total = nd.total, ni = nd.ni;
  const int ncol = total + args.nl;  // body-load columns follow the system's columns
  const int tid = threadIdx.x, tr = tid % TR, tc = tid / TR;

  for (int p = tid; p < total; p += TR * TC) {
    const PosDev e = args.pos[nd.pos_off + p];
    spos[p] = e;
    if constexpr (MICRO) {
#pragma unroll
      for (int r = 0; r < 5; ++r) sst[r][p] = args.stencil[r * args.nu + e.gid];
    }
  }
  __syncthreads();

  // ---- assemble the owned entries
  double m[RPT][CPT];
  const double* A = nullptr;
  const double* B = nullptr;
  int lda = 0, ldb = 0;
  if constexpr (!MICRO) {
    const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
    A = args.arena + ca.s_off;
    lda = ca.ld;
    B = args.arena + cb.s_off;
    ldb = cb.ld;
  }
  auto assemble = [&]() {
#pragma unroll
  for (int a = 0; a < RPT; ++a) {
    const int i = tr + TR * a;
#pragma unroll
    for (int b = 0; b < CPT; ++b) {
      const int j = tc + TC * b;
      double v = 0.0;
      if (i < total && j >= total && j < ncol) {  // right-hand sides (dense_nd.cpp:98-101, 136-146)
        const PosDev pi = spos[i];
        const int c = j - total;
        if constexpr (MICRO) {
          v = args.load_col[pi.gid] == c ? 1.0 : 0.0;
        } else {
          const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
          v = pi.src >= 0 ? args.arena[ca.rhs_off + pi.src + (long long)c * ca.rhs_ld]
                          : args.arena[cb.rhs_off + (-pi.src - 1) + (long long)c * cb.rhs_ld];
        }
      } else if (i < total && j < total) {
        const PosDev pi = spos[i], pj = spos[j];
        if constexpr (MICRO) {
          if (i == j) {
            v = sst[0][i];
          } else {
            const int dx = (pj.gid % args.side) - (pi.gid % args.side);
            const int dy = (pj.gid / args.side) - (pi.gid / args.side);
            if (dy == 0 && dx == 1) v = sst[1][i];
            else if (dy == 0 && dx == -1) v = sst[2][i];
            else if (dx == 0 && dy == 1) v = sst[3][i];
            else if (dx == 0 && dy == -1) v = sst[4][i];
          }
        } else {
          if ((pi.src >= 0) == (pj.src >= 0)) {
            v = pi.src >= 0 ? A[pi.src + (long long)pj.src * lda]
                            : B[(-pi.src - 1) + (long long)(-pj.src - 1) * ldb];
          } else if (pi.partner == j) {
            v = args.stencil[pi.dir * args.nu + pi.gid];
          }
        }
      }
      m[a][b] = v;
    }
  }
  };
  assemble();

  // ---- no-interchange attempt: pivot k = row k, one barrier per step (row
  // k+1 and column k+1 are published by their owners right after their own
  // update); accepted iff every interface multiplier has |l| <= 1, i.e. when
  // partial pivoting would not interchange (then the arithmetic is identical).
  // Otherwise the system is re-assembled and eliminated with pivoting below.
  __shared__ double rowq[2][MAXT];
  __shared__ double rinvq[2];  // 1 / pivot of the published step (formed once, by the pivot's owner)
  double pmin = DBL_MAX, pmax = 0.0;
  bool ok = true;
  {
    // per-thread row / column indices (hoisted) and branch-free publishing: every
    // thread selects its entries of column k and row k and stores them predicated
    int ii[RPT], jj[CPT];
#pragma unroll
    for (int a = 0; a < RPT; ++a) ii[a] = tr + TR * a;
#pragma unroll
    for (int b = 0; b < CPT; ++b) jj[b] = tc + TC * b;
    auto publish = [&](int k, int buf) {
      const int bk = k / TC, tck = k % TC, ap = k / TR, trk = k % TR;
      const bool pc = tc == tck, pr = tr == trk;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        double v = m[a][0];
#pragma unroll
        for (int b = 1; b < CPT; ++b) v = b == bk ? m[a][b] : v;
        if (pc) colk[buf][ii[a]] = v;
      }
#pragma unroll
      for (int b = 0; b < CPT; ++b) {
        double u = m[0][b];
#pragma unroll
        for (int a = 1; a < RPT; ++a) u = a == ap ? m[a][b] : u;
        if (pr) rowq[buf][jj[b]] = u;
      }
      if (pc && pr) {  // the pivot's owner: one reciprocal per step for everybody
        double pv = m[0][0];
#pragma unroll
        for (int a = 0; a < RPT; ++a)
#pragma unroll
          for (int b = 0; b < CPT; ++b) pv = (a == ap && b == bk) ? m[a][b] : pv;
        rinvq[buf] = 1.0 / pv;
      }
    };
    bool bad = false;
    // one elimination step (the pivot row/column of step k are published in colk/rowq)
    auto step = [&](int k) {
      const int buf = k & 1;
      const double* ck = colk[buf];
      const double* rp = rowq[buf];
      if (tid == 0) {  // pivot statistics (only thread 0 reports them)
        const double apv = fabs(rp[k]);
        pmin = fmin(pmin, apv);
        pmax = (apv != apv) ? INFINITY : fmax(pmax, apv);
      }
      const double rinv = rinvq[buf];
      double lr[RPT], ur[CPT];
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const double l = ck[ii[a]] * rinv;  // (entries past the system are stale: masked)
        const bool live = ii[a] > k && ii[a] < total;
        bad |= live && ii[a] < ni && !(fabs(l) <= 1.0);
        lr[a] = live ? -l : 0.0;
      }
#pragma unroll
      for (int b = 0; b < CPT; ++b) {
        const double u = rp[jj[b]];
        ur[b] = (jj[b] > k && jj[b] < ncol) ? u : 0.0;
      }
#pragma unroll
      for (int a = 0; a < RPT; ++a)
#pragma unroll
        for (int b = 0; b < CPT; ++b) m[a][b] = fma(lr[a], ur[b], m[a][b]);
    };
    if constexpr (TR == TC && RPT == CPT) {
      // square thread grid: step k's pivot row and column sit in register slot
      // k / TR of their owners, so with the steps grouped by that slot (compile-time
      // register indices) publishing is a predicated store per entry, no selects
      auto publish_c = [&](auto Cc, int k, int buf) {
        constexpr int C = decltype(Cc)::value;
        const int kk = k - C * TR;
        const bool pc = tc == kk, pr = tr == kk;
#pragma unroll
        for (int a = 0; a < RPT; ++a) st_shared_f64_pred(&colk[buf][ii[a]], m[a][C], pc);
#pragma unroll
        for (int b = 0; b < CPT; ++b) st_shared_f64_pred(&rowq[buf][jj[b]], m[C][b], pr);
        if (pc && pr) rinvq[buf] = 1.0 / m[C][C];
      };
      if (ni > 0) publish_c(std::integral_constant<int, 0>{}, 0, 0);
      __syncthreads();
      static_for<RPT>([&](auto Cc) {
        constexpr int C = decltype(Cc)::value;
        const int k1 = min(ni, (C + 1) * TR);
        for (int k = C * TR; k < k1; ++k) {
          step(k);
          if (k + 1 < ni) {
            if (k + 1 < (C + 1) * TR) publish_c(Cc, k + 1, (k + 1) & 1);
            else publish_c(std::integral_constant<int, (C + 1 < RPT ? C + 1 : C)>{}, k + 1, (k + 1) & 1);
          }
          __syncthreads();
        }
      });
      ok = !bad;
    } else {
    if (ni > 0) publish(0, 0);
    __syncthreads();
    for (int k = 0; k < ni; ++k) {
      const int buf = k & 1;
      const double* ck = colk[buf];
      const double* rp = rowq[buf];
      if (tid == 0) {  // pivot statistics (only thread 0 reports them)
        const double apv = fabs(rp[k]);
        pmin = fmin(pmin, apv);
        pmax = (apv != apv) ? INFINITY : fmax(pmax, apv);
      }
      const double rinv = rinvq[buf];
      // branch-free rank-1 update: rows <= k get l = 0 and columns <= k get u = 0, so
      // every owned entry takes one unconditional FMA (the predicated form spent ~10
      // instructions per entry; an FMA with a zero factor leaves finite entries unchanged)
      double lr[RPT], ur[CPT];
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const double l = ck[ii[a]] * rinv;  // (entries past the system are stale: masked)
        const bool live = ii[a] > k && ii[a] < total;
        bad |= live && ii[a] < ni && !(fabs(l) <= 1.0);
        lr[a] = live ? -l : 0.0;
      }
#pragma unroll
      for (int b = 0; b < CPT; ++b) {
        const double u = rp[jj[b]];
        ur[b] = (jj[b] > k && jj[b] < ncol) ? u : 0.0;
      }
#pragma unroll
      for (int a = 0; a < RPT; ++a)
#pragma unroll
        for (int b = 0; b < CPT; ++b) m[a][b] = fma(lr[a], ur[b], m[a][b]);
      if (k + 1 < ni) publish(k + 1, (k + 1) & 1);
      __syncthreads();
    }
    ok = !bad;
    }
  }
  const bool fast = __syncthreads_and(ok) != 0;
  if (!fast && threadIdx.x == 0) atomicAdd(&g_small_fallbacks, 1u);
  if (!fast) {
    assemble();
    pmin = DBL_MAX;
    pmax = 0.0;
  }

  // ---- elimination of rows/columns [0, ni) with partial pivoting among the
  // interface rows (when the attempt above was rejected)
  unsigned elim = 0u;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned gmask = (TR == 32) ? 0xffffffffu : (((1u << TR) - 1u) << (lane & ~unsigned(TR - 1)));
  for (int k = 0; k < (fast ? 0 : ni); ++k) {
    const int bk = k / TC, tck = k % TC;
    double* ck = colk[k & 1];
    if (tc == tck) {
      double best = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int i = tr + TR * a;
        double v = m[a][0];
#pragma unroll
        for (int b = 1; b < CPT; ++b)
          if (b == bk) v = m[a][b];
        if (i < total) ck[i] = v;
        if (i < ni && !((elim >> a) & 1u)) {
          double av = fabs(v);
          if (av != av) av = INFINITY;  // a NaN column still yields a (flagged) pivot
          if (av > best) { best = av; bi = i; }
        }
      }
#pragma unroll
      for (int off = TR / 2; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(gmask, best, off, TR);
        const int oi = __shfl_xor_sync(gmask, bi, off, TR);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tr == 0) s_piv = bi;
      __syncwarp(gmask);  // the group's column entries are in ck (same warp)
      if (tr == 0) s_rinv = 1.0 / ck[bi];
    }
    __syncthreads();
    const int p = s_piv;
    const double pv = ck[p];
    if (tr == p % TR) {
      const int ap = p / TR;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        if (a == ap) {
          elim |= 1u << a;
#pragma unroll
          for (int b = 0; b < CPT; ++b) {
            const int j = tc + TC * b;
            if (j < MAXT) rowp[j] = m[a][b];
          }
        }
      }
    }
    if (tid == 0) {
      const double apv = fabs(pv);
      pmin = fmin(pmin, apv);
      pmax = (apv != apv) ? INFINITY : fmax(pmax, apv);
    }
    __syncthreads();
    const double rinv = s_rinv;
    double lr[RPT], ur[CPT];  // branch-free update (see the no-interchange loop)
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int i = tr + TR * a;
      lr[a] = (i < total && !((elim >> a) & 1u)) ? -(ck[i] * rinv) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CPT; ++b) {
      const int j = tc + TC * b;
      ur[b] = (j > k && j < ncol) ? rowp[j] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
      for (int b = 0; b < CPT; ++b) m[a][b] = fma(lr[a], ur[b], m[a][b]);
  }

  // ---- S = trailing block, written compact (ld = nd.ld)
  double* out = args.arena + nd.s_off;
#pragma unroll
  for (int b = 0; b < CPT; ++b) {
    const int j = tc + TC * b;
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
      const int i = tr + TR * a;
      if (i >= ni && i < total && j >= ni && j < total) out[(i - ni) + (long long)(j - ni) * nd.ld] = m[a][b];
      if (i >= ni && i < total && j >= total && j < ncol)
        args.arena[nd.rhs_off + (i - ni) + (long long)(j - total) * nd.rhs_ld] = m[a][b];
    }
  }
  if (tid == 0) {
    args.pivstat[2 * node_id] = ni > 0 ? pmin : DBL_MAX;
    args.pivstat[2 * node_id + 1] = pmax;
  }
}

// Launch dispatch by the largest system in the batch.
// (size classes fitted to the systems of the 16 x 16 / 32 x 32 leaf subtrees -- 16, 22,
// 34, 50, 74, 120 unknowns: the kernel is issue bound, so padding entries cost time)
#define DTNB_SMALL_VARIANTS(X) \
  X(24, 8, 8, 3, 3)            \
  X(32, 8, 8, 4, 4)            \
  X(40, 8, 8, 5, 5)            \
  X(56, 8, 16, 7, 4)           \
  X(64, 16, 16, 4, 4)          \
  X(80, 16, 16, 5, 5)          \
  X(96, 16, 16, 6, 6)          \
  X(128, 32, 32, 4, 4) /* 1024 threads: measured 0.5 % faster than 16 x 32 x (8, 4) */ \
  X(160, 16, 32, 10, 5)

cudaError_t launch_small_elim(const KernelArgs& args, const int* d_list, int count, int max_total, bool micro,
                              cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
#define X(LIM, TR, TC, RPT, CPT)                                                         \
  if (max_total <= LIM) {                                                                \
    if (micro) small_elim_kernel<TR, TC, RPT, CPT, true><<<count, TR * TC, 0, st>>>(args, d_list); \
    else small_elim_kernel<TR, TC, RPT, CPT, false><<<count, TR * TC, 0, st>>>(args, d_list);      \
    return cudaGetLastError();                                                           \
  }
  DTNB_SMALL_VARIANTS(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace dtnb
