// One-CTA fused merge for the many-system waves around the reference leaves (merge_two,
// dense_nd.cpp:105-186, on systems of 28..64 interface unknowns and up to ~190 boundary
// unknowns): the whole merge -- assembly from the two children's Schur complements and
// the cross-interface stencil couplings (dense_nd.cpp:114-165), PartialPivLU of the
// interface block (dense_nd.cpp:174), X = M_ii^{-1} M_ib, S = M_bb - M_bi X
// (dense_nd.cpp:181, the reference's association) -- runs in ONE launch with the system in
// shared memory, instead of gather + panels + row panels + trailing updates + substitution
// + Schur GEMM launches on an HBM-resident system (or, below 160 unknowns, rank-1 updates
// of the whole total x total system in registers with ~7 % of the issue slots doing FP64).
//
// Shared memory: T = [M_ii | M_ib] (ni x total, column-major, leading dimension LDT == 2 mod 16
// doubles: 16-byte column accesses of consecutive columns are bank-conflict free) and
// M_bi (nb x ni). M_bb never enters shared memory: it is gathered from the children straight
// into the accumulators of the Schur-complement tiles.
//   LU: thread j owns column j; per pivot step warp 0 finds the pivot (largest |a|, ties to
//     the lowest row: partial pivoting among the interface rows) and publishes the
//     multipliers, then every column swaps its two entries and takes the rank-1 update
//     (two barriers per step; columns of M_ib ride along, so Y = L^{-1} P M_ib needs no L).
//   X = U^{-1} Y: one thread per boundary column, column-oriented back substitution.
//   S = M_bb - M_bi X: FP64 tensor cores (DMMA m16n8k4), 32 x 32 output blocks per warp; the
//     MMA's logical rows (g, g + 8) are the adjacent rows (2g, 2g + 1) of M_bi and its logical
//     k index t of two consecutive k steps is the physical (2t, 2t + 1), so every fragment
//     is one 16-byte shared load (as in k_tma.cu).
#include <cfloat>

#include "common.cuh"

namespace dtnb {

constexpr int FNT = 256;  // threads per CTA (one per system column in the LU)
constexpr int FKB = 8;    // pivots per LU block / rows per substitution block

struct FusedShape {  // shared-memory carve-up of one launch (host and device agree through these)
  int ldt, tcols, ldb, kpad;
  size_t bytes;
};
__host__ __device__ inline FusedShape fused_shape(int max_ni, int max_nb, int max_total) {
  FusedShape s;
  s.ldt = max_ni <= 32 ? 34 : 66;
  s.kpad = (max_ni + 7) & ~7;                   // k extent of the Schur GEMM (zero padded)
  s.tcols = max_ni + ((max_nb + 31) & ~31);     // B fragments of ragged blocks stay inside T
  s.ldb = ((max_nb + 31) & ~31) + 2;            // A fragments likewise
  s.bytes = size_t(max_total) * sizeof(PosDev) + (size_t(s.ldt) * s.tcols + size_t(s.ldb) * s.kpad + 64 * FKB + 64) * 8 + 64;
  return s;
}

// phase clocks of CTA 0 of the last launch of each size class (diagnostic, dtn_debug_fused_clocks)
__device__ long long g_fused_clk[3][8];
#define FCLK(slot) do { if (blockIdx.x == 0 && tid == 0) g_fused_clk[fcls][slot] = clock64(); } while (0)

__device__ __forceinline__ double2 f_lds128(const double* p) {  // (a plain load: ordered with the C++ stores)
  return *reinterpret_cast<const double2*>(p);
}

__global__ void __launch_bounds__(FNT, 2) fused_merge_kernel(KernelArgs args, const int* __restrict__ list, int max_ni,
                                                          int max_nb, int max_total) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  const FusedShape sh = fused_shape(max_ni, max_nb, max_total);
  PosDev* spos = reinterpret_cast<PosDev*>(fsm_raw);
  double* T = reinterpret_cast<double*>(fsm_raw + ((size_t(max_total) * sizeof(PosDev) + 15) & ~size_t(15)));
  double* Mbi = T + size_t(sh.ldt) * sh.tcols;
  double* lpan = Mbi + size_t(sh.ldb) * sh.kpad;  // [64][FKB] multipliers of the current LU block
  double* urinv = lpan + 64 * FKB;
  __shared__ int s_pv[FKB];
  const int LDT = sh.ldt, LDB = sh.ldb;

  const int node_id = list[blockIdx.x];
  const NodeDev nd = args.nodes[node_id];
  const int total = nd.total, ni = nd.ni, nb = total - ni;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* __restrict__ A = args.arena + ca.s_off;
  const double* __restrict__ B = args.arena + cb.s_off;
  const long long lda = ca.ld, ldb_ = cb.ld;
  double* S = args.arena + nd.s_off;  // (written here, read back by this CTA only: plain loads)
  const long long lds = nd.ld;
  // entry (i, j) of the merge system (dense_nd.cpp:114-165 as a gather): its address, or null for 0
  auto entry_ptr = [&](const PosDev& pi, const PosDev& pj, int j) -> const double* {
    if ((pi.src >= 0) == (pj.src >= 0))
      return pi.src >= 0 ? A + (pi.src + (long long)pj.src * lda) : B + ((-pi.src - 1) + (long long)(-pj.src - 1) * ldb_);
    if (pi.partner == j) return args.stencil + (pi.dir * args.nu + pi.gid);
    return nullptr;
  };
  const int fcls = max_ni > 32 ? 2 : (max_nb > 64 ? 1 : 0);
  FCLK(0);
  for (int p = tid; p < total; p += FNT) spos[p] = args.pos[nd.pos_off + p];
  if (tid < 64) urinv[tid] = 0.0;
  __syncthreads();
  // ---- assembly: T = [M_ii | M_ib] (rows [ni, kpad) zero: the Schur GEMM's k padding), M_bi.
  // Batches of GB independent gathers per thread: addresses first, then the loads in
  // flight together, then the shared stores (a store between two loads would serialise them)
  const int kpad = (ni + 7) & ~7;
  {
    // warps over columns, lanes over rows (consecutive rows of one child are consecutive
    // addresses); 8 independent gathers per thread in flight, no integer divisions
    const int nh = (kpad + 31) >> 5;  // row chunks of 32 (kpad = 8 .. 64)
    for (int jb = warp * 4; jb < total; jb += 4 * (FNT / 32)) {
      const double* ptr[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = jb + q;
        const PosDev pj = spos[min(j, total - 1)];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 32 * h;
          ptr[q][h] = (j < total && h < nh && i < ni) ? entry_ptr(spos[i], pj, j) : nullptr;
        }
      }
      double v[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) v[q][h] = ptr[q][h] ? __ldg(ptr[q][h]) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 32 * h, j = jb + q;
          if (j < total && i < kpad) T[i + j * LDT] = v[q][h];
        }
    }
    // M_bi (columns [0, kpad)) into shared memory, M_bb (columns [0, nb)) straight into S
    // (global): the Schur GEMM starts from it
    for (int pass = 0; pass < 2; ++pass) {
      const int ncol = pass == 0 ? kpad : nb;
      for (int rb = 0; rb < nb; rb += 128)
        for (int cb = warp * 2; cb < ncol; cb += 2 * (FNT / 32)) {
          const double* ptr[2][4];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = cb + q;
            const bool cok = c < (pass == 0 ? ni : nb);
            const int cs = pass == 0 ? c : ni + c;  // system column
            const PosDev pc = spos[cok ? cs : 0];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int r = rb + lane + 32 * h;
              ptr[q][h] = (cok && r < nb) ? entry_ptr(spos[ni + r], pc, cs) : nullptr;
            }
          }
          double v[2][4];
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int h = 0; h < 4; ++h) v[q][h] = ptr[q][h] ? __ldg(ptr[q][h]) : 0.0;
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int r = rb + lane + 32 * h, c = cb + q;
              if (c < ncol && r < nb) {
                if (pass == 0) Mbi[r + c * LDB] = v[q][h];
                else S[r + (long long)c * lds] = v[q][h];
              }
            }
        }
    }
  }
  __syncthreads();
  FCLK(1);
  // ---- blocked LU of the ni interface rows (partial pivoting), blocks of FKB = 8 pivots.
  // A rank-1 update per pivot would stream the whole trailing block through shared memory
  // at every step (measured: 1300-2000 cycles per pivot). Instead warp 0 factors the
  // block's 8 columns in REGISTERS (lane = row, rows lane and lane + 32; pivot search by
  // warp reductions, row exchanges by shuffles, no barriers), publishes the multipliers
  // (lpan, one 64-byte row per system row) and the pivot rows, and then every other column
  // applies the 8 row exchanges, solves its 8 entries of U12 / Y against the unit-lower
  // L11 and takes ONE rank-8 update: each trailing entry is loaded and stored once per 8 pivots.
  double pmin = DBL_MAX, pmax = 0.0;
  long long fq = clock64(), fpan = 0, fupd = 0;
  for (int k0 = 0; k0 < ni; k0 += FKB) {
    const int kb = min(FKB, ni - k0);
    if (warp == 0) {
      const int r0 = lane, r1 = lane + 32;
      double v0[FKB], v1[FKB];
#pragma unroll
      for (int q = 0; q < FKB; ++q) {
        v0[q] = (q < kb && r0 < ni) ? T[r0 + (k0 + q) * LDT] : 0.0;
        v1[q] = (q < kb && r1 < ni) ? T[r1 + (k0 + q) * LDT] : 0.0;
      }
      // no-interchange attempt (as the other LU kernels): eliminate with pivot k = row k and
      // accept iff every multiplier has |l| <= 1, i.e. iff partial pivoting would not
      // interchange (ties go to the lowest row, which is row k) -- then the arithmetic is
      // the pivoted elimination's, without the pivot search and the row exchanges
      bool fast;
      {
        const bool khi = k0 >= 32;  // (a block of 8 never straddles row 32)
        bool bad = false;
        double rv[FKB], pvv[FKB];
#pragma unroll
        for (int sidx = 0; sidx < FKB; ++sidx) {
          if (sidx < kb) {
            const int k = k0 + sidx;
            double xp[FKB];
#pragma unroll
            for (int q = sidx; q < FKB; ++q) xp[q] = __shfl_sync(0xffffffffu, khi ? v1[q] : v0[q], k & 31);
            const double rinv = 1.0 / xp[sidx];
            rv[sidx] = rinv;
            pvv[sidx] = xp[sidx];
            bad |= !(fabs(xp[sidx]) > 0.0) || fabs(xp[sidx]) == INFINITY;  // zero / NaN / inf pivot: pivoted path
            if (r0 > k && r0 < ni) {
              const double l = v0[sidx] * rinv;
              bad |= !(fabs(l) <= 1.0);
              v0[sidx] = l;
#pragma unroll
              for (int q = sidx + 1; q < FKB; ++q) v0[q] = fma(-l, xp[q], v0[q]);
            }
            if (r1 > k && r1 < ni) {
              const double l = v1[sidx] * rinv;
              bad |= !(fabs(l) <= 1.0);
              v1[sidx] = l;
#pragma unroll
              for (int q = sidx + 1; q < FKB; ++q) v1[q] = fma(-l, xp[q], v1[q]);
            }
          }
        }
        fast = !__any_sync(0xffffffffu, bad);
        if (fast) {
          if (lane < kb) s_pv[lane] = k0 + lane;
#pragma unroll
          for (int sidx = 0; sidx < FKB; ++sidx)
            if (sidx < kb && lane == 0) {
              urinv[k0 + sidx] = rv[sidx];
              const double apv = fabs(pvv[sidx]);
              pmin = fmin(pmin, apv);
              pmax = fmax(pmax, apv);
            }
        } else {  // restart from the block's columns as the previous blocks left them
#pragma unroll
          for (int q = 0; q < FKB; ++q) {
            v0[q] = (q < kb && r0 < ni) ? T[r0 + (k0 + q) * LDT] : 0.0;
            v1[q] = (q < kb && r1 < ni) ? T[r1 + (k0 + q) * LDT] : 0.0;
          }
        }
      }
#pragma unroll
      for (int sidx = 0; sidx < FKB; ++sidx) {
        if (sidx < kb && !fast) {  // (uniform)
          const int k = k0 + sidx;
          const double a0 = (r0 >= k && r0 < ni) ? fabs(v0[sidx]) : -1.0;
          const double a1 = (r1 >= k && r1 < ni) ? fabs(v1[sidx]) : -1.0;
          // |a| as ordered bits (a NaN sorts above inf: a NaN column still yields a flagged pivot)
          const bool nan0 = a0 != a0, nan1 = a1 != a1;
          const bool take1 = (a1 >= 0.0 || nan1) && !nan0 && (a0 < 0.0 || nan1 || a1 > a0);
          const double av = take1 ? a1 : a0;
          const int ar = take1 ? r1 : r0;
          const unsigned hi = (av >= 0.0 || av != av) ? (unsigned(__double2hiint(av)) | 0x80000000u) : 0u;
          const unsigned lo = unsigned(__double2loint(av));
          const unsigned whi = __reduce_max_sync(0xffffffffu, hi);
          const unsigned wlo = __reduce_max_sync(0xffffffffu, hi == whi ? lo : 0u);
          const int p = int(__reduce_min_sync(0xffffffffu, (hi == whi && lo == wlo) ? unsigned(ar) : 0xffffffffu));
          // exchange rows k and p of the panel (all 8 columns: L stays in the final row order)
          const bool k_hi = k >= 32, p_hi = p >= 32;
          const bool own_k = (k_hi ? r1 : r0) == k, own_p = (p_hi ? r1 : r0) == p;
          double xp[FKB];
#pragma unroll
          for (int q = 0; q < FKB; ++q) {
            const double xk = __shfl_sync(0xffffffffu, k_hi ? v1[q] : v0[q], k & 31);
            xp[q] = __shfl_sync(0xffffffffu, p_hi ? v1[q] : v0[q], p & 31);
            if (own_p) {
              if (p_hi) v1[q] = xk;
              else v0[q] = xk;
            }
            if (own_k) {  // (after own_p: for p == k the row keeps its values)
              if (k_hi) v1[q] = xp[q];
              else v0[q] = xp[q];
            }
          }
          const double piv = xp[sidx];
          const double rinv = 1.0 / piv;
          if (lane == 0) {
            s_pv[sidx] = p;
            urinv[k] = rinv;
            const double apv = fabs(piv);
            pmin = fmin(pmin, apv);
            pmax = (apv != apv) ? INFINITY : fmax(pmax, apv);
          }
          if (r0 > k && r0 < ni) {
            const double l = v0[sidx] * rinv;
            v0[sidx] = l;
#pragma unroll
            for (int q = sidx + 1; q < FKB; ++q) v0[q] = fma(-l, xp[q], v0[q]);
          }
          if (r1 > k && r1 < ni) {
            const double l = v1[sidx] * rinv;
            v1[sidx] = l;
#pragma unroll
            for (int q = sidx + 1; q < FKB; ++q) v1[q] = fma(-l, xp[q], v1[q]);
          }
        }
      }
      // publish: the factored panel back into T (U11 for the substitution) and the multiplier
      // rows (rows [ni, 64): zero, they pad the rank-8 update)
#pragma unroll
      for (int q = 0; q < FKB; ++q) {
        if (q < kb && r0 >= k0 && r0 < ni) T[r0 + (k0 + q) * LDT] = v0[q];
        if (q < kb && r1 >= k0 && r1 < ni) T[r1 + (k0 + q) * LDT] = v1[q];
      }
#pragma unroll
      for (int q = 0; q < FKB; q += 2) {
        *reinterpret_cast<double2*>(lpan + r0 * FKB + q) = make_double2(v0[q], v0[q + 1]);
        *reinterpret_cast<double2*>(lpan + r1 * FKB + q) = make_double2(v1[q], v1[q + 1]);
      }
    }
    { const long long n_ = clock64(); fpan += n_ - fq; fq = n_; }
    __syncthreads();
    if (tid >= k0 + kb && tid < total) {
      double* cj = T + tid * LDT;
      for (int sidx = 0; sidx < kb; ++sidx) {  // the block's row exchanges, in order
        const int p = s_pv[sidx], k = k0 + sidx;
        const double a = cj[k], b = cj[p];
        cj[p] = a;
        cj[k] = b;
      }
      double u[FKB];
#pragma unroll
      for (int q = 0; q < FKB; q += 2) {
        const double2 t = f_lds128(cj + k0 + q);
        u[q] = t.x;
        u[q + 1] = t.y;
      }
      // u <- L11^{-1} u (unit lower; rows past kb have zero multipliers)
#pragma unroll
      for (int t = 1; t < FKB; ++t) {
        double lr[FKB];
#pragma unroll
        for (int q = 0; q < FKB; q += 2) {
          const double2 l2 = f_lds128(lpan + (k0 + t) * FKB + q);
          lr[q] = l2.x;
          lr[q + 1] = l2.y;
        }
#pragma unroll
        for (int q = 0; q < t; ++q) u[t] = fma(-lr[q], u[q], u[t]);
      }
#pragma unroll
      for (int q = 0; q < FKB; q += 2) *reinterpret_cast<double2*>(cj + k0 + q) = make_double2(u[q], u[q + 1]);
      // rank-8 update of the rows below the block, two row pairs per iteration
      for (int i = k0 + FKB; i < kpad; i += 4) {
        double2 c0 = f_lds128(cj + i), c1 = f_lds128(cj + i + 2);
        double2 la[4], lb[4], lc[4], ld[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          la[q] = f_lds128(lpan + (i + 0) * FKB + 2 * q);
          lb[q] = f_lds128(lpan + (i + 1) * FKB + 2 * q);
          lc[q] = f_lds128(lpan + (i + 2) * FKB + 2 * q);
          ld[q] = f_lds128(lpan + (i + 3) * FKB + 2 * q);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          c0.x = fma(-la[q].x, u[2 * q], c0.x);
          c0.x = fma(-la[q].y, u[2 * q + 1], c0.x);
          c0.y = fma(-lb[q].x, u[2 * q], c0.y);
          c0.y = fma(-lb[q].y, u[2 * q + 1], c0.y);
          c1.x = fma(-lc[q].x, u[2 * q], c1.x);
          c1.x = fma(-lc[q].y, u[2 * q + 1], c1.x);
          c1.y = fma(-ld[q].x, u[2 * q], c1.y);
          c1.y = fma(-ld[q].y, u[2 * q + 1], c1.y);
        }
        *reinterpret_cast<double2*>(cj + i) = c0;
        *reinterpret_cast<double2*>(cj + i + 2) = c1;
      }
    }
    __syncthreads();
    { const long long n_ = clock64(); fupd += n_ - fq; fq = n_; }
  }
  FCLK(2);
  if (blockIdx.x == 0 && tid == 0) { g_fused_clk[fcls][5] = fpan; g_fused_clk[fcls][6] = fupd; }
  // ---- X = U^{-1} Y, one boundary column per thread, blocks of 8 rows from the bottom: the
  // block's 8 unknowns live in registers, the rows above take one rank-8 update per block
  // (padding rows [ni, kpad): zero entries and urinv = 0 give x = 0)
  if (tid >= ni && tid < total) {
    double* cj = T + tid * LDT;
    for (int r0 = kpad - FKB; r0 >= 0; r0 -= FKB) {
      double x[FKB];
#pragma unroll
      for (int q = 0; q < FKB; q += 2) {
        const double2 t = f_lds128(cj + r0 + q);
        x[q] = t.x;
        x[q + 1] = t.y;
      }
#pragma unroll
      for (int q = FKB - 1; q >= 0; --q) {
        const double* uc = T + (r0 + q) * LDT + r0;  // U[r0 .. r0 + q][r0 + q]
        x[q] *= urinv[r0 + q];
        double ut[FKB];
#pragma unroll
        for (int t = 0; t < FKB; t += 2) {
          if (t < q) {
            const double2 t2 = f_lds128(uc + t);
            ut[t] = t2.x;
            ut[t + 1] = t2.y;
          }
        }
#pragma unroll
        for (int t = 0; t < q; ++t) x[t] = fma(-ut[t], x[q], x[t]);
      }
#pragma unroll
      for (int q = 0; q < FKB; q += 2) *reinterpret_cast<double2*>(cj + r0 + q) = make_double2(x[q], x[q + 1]);
      for (int i = 0; i < r0; i += 4) {
        double2 c0 = f_lds128(cj + i), c1 = f_lds128(cj + i + 2);
        double2 ua[FKB], ub[FKB];
#pragma unroll
        for (int q = 0; q < FKB; ++q) {
          ua[q] = f_lds128(T + (r0 + q) * LDT + i);
          ub[q] = f_lds128(T + (r0 + q) * LDT + i + 2);
        }
#pragma unroll
        for (int q = 0; q < FKB; ++q) {
          c0.x = fma(-ua[q].x, x[q], c0.x);
          c0.y = fma(-ua[q].y, x[q], c0.y);
          c1.x = fma(-ub[q].x, x[q], c1.x);
          c1.y = fma(-ub[q].y, x[q], c1.y);
        }
        *reinterpret_cast<double2*>(cj + i) = c0;
        *reinterpret_cast<double2*>(cj + i + 2) = c1;
      }
    }
  }
  __syncthreads();
  FCLK(3);
  // ---- S = M_bb - M_bi X on the FP64 tensor cores, 32 x 16 output blocks round-robin over
  // the warps; M_bb was gathered into S by the assembly pass (it initialises the accumulators)
  const int g = lane >> 2, tig = lane & 3;
  const int nbm = (nb + 31) >> 5, nbn = (nb + 15) >> 4;
  for (int blk = warp; blk < nbm * nbn; blk += FNT / 32) {
    const int r0 = (blk % nbm) * 32, c0 = (blk / nbm) * 16;
    double acc[2][2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = r0 + i * 16 + 2 * g + (v >> 1);
          const int c = c0 + jn * 8 + 2 * tig + (v & 1);
          acc[i][jn][v] = (r < nb && c < nb) ? -S[r + c * lds] : 0.0;  // -M_bb
        }
    const double* ab = Mbi + r0 + 2 * g;
    const double* bb = T + (ni + c0 + g) * LDT + 2 * tig;
    for (int k8 = 0; k8 < kpad; k8 += 8) {
      double2 af[2][2], bf[2];
#pragma unroll
      for (int st = 0; st < 2; ++st)
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i][st] = f_lds128(ab + i * 16 + (k8 + 2 * tig + st) * LDB);
#pragma unroll
      for (int jn = 0; jn < 2; ++jn) bf[jn] = f_lds128(bb + jn * 8 * LDT + k8);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jn = 0; jn < 2; ++jn) {
          mma_f64_m16n8k4(acc[i][jn], af[i][0].x, af[i][0].y, bf[jn].x);
          mma_f64_m16n8k4(acc[i][jn], af[i][1].x, af[i][1].y, bf[jn].y);
        }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 2; ++jn)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int r = r0 + i * 16 + 2 * g + (v >> 1);
          const int c = c0 + jn * 8 + 2 * tig + (v & 1);
          if (r < nb && c < nb) S[r + c * lds] = -acc[i][jn][v];
        }
  }
  FCLK(4);
  if (tid == 0) {
    args.pivstat[2 * node_id] = ni > 0 ? pmin : DBL_MAX;
    args.pivstat[2 * node_id + 1] = pmax;
  }
}

// Largest dynamic shared memory a launch may ask for (set once per device by fused_init)
constexpr size_t FUSED_SMEM_MAX = 220 * 1024;

void fused_clocks_read(long long* out24) { cudaMemcpyFromSymbol(out24, g_fused_clk, sizeof(long long) * 24); }

cudaError_t fused_init() {
  return cudaFuncSetAttribute(fused_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(FUSED_SMEM_MAX));
}

// A wave of merges can take the fused kernel when its largest system fits one CTA's shared memory.
bool fused_merge_fits(int max_ni, int max_nb, int max_total) {
  if (max_ni < 1 || max_ni > 64 || max_total > FNT || max_nb < 1) return false;
  return fused_shape(max_ni, max_nb, max_total).bytes <= FUSED_SMEM_MAX;
}

cudaError_t launch_fused_merge(const KernelArgs& args, const int* d_list, int count, int max_ni, int max_nb,
                               int max_total, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const FusedShape s = fused_shape(max_ni, max_nb, max_total);
  fused_merge_kernel<<<count, FNT, s.bytes, st>>>(args, d_list, max_ni, max_nb, max_total);
  return cudaGetLastError();
}

}  // namespace dtnb
