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
  s.bytes = size_t(max_total) * sizeof(PosDev) + (size_t(s.ldt) * s.tcols + size_t(s.ldb) * s.kpad + 2 * 64) * 8 + 64;
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
  double* lvec = Mbi + size_t(sh.ldb) * sh.kpad;
  double* urinv = lvec + 64;
  __shared__ int s_piv;
  const int LDT = sh.ldt, LDB = sh.ldb;

  const int node_id = list[blockIdx.x];
  const NodeDev nd = args.nodes[node_id];
  const int total = nd.total, ni = nd.ni, nb = total - ni;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const NodeDev ca = args.nodes[nd.a], cb = args.nodes[nd.b];
  const double* __restrict__ A = args.arena + ca.s_off;
  const double* __restrict__ B = args.arena + cb.s_off;
  const long long lda = ca.ld, ldb_ = cb.ld;
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
  if (tid < 64) lvec[tid] = 0.0;
  __syncthreads();
  // ---- assembly: T = [M_ii | M_ib] (rows [ni, kpad) zero: the Schur GEMM's k padding), M_bi.
  // Batches of GB independent gathers per thread: addresses first, then the loads in
  // flight together, then the shared stores (a store between two loads would serialise them)
  const int kpad = (ni + 7) & ~7;
  constexpr int GB = 8;
  {
    const int nT = kpad * total;  // element e: row e % kpad of column e / kpad
    for (int e0 = tid; e0 < nT; e0 += GB * FNT) {
      const double* ptr[GB];
      double v[GB];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int e = e0 + q * FNT;
        const int i = e % kpad, j = e / kpad;
        ptr[q] = (e < nT && i < ni) ? entry_ptr(spos[i], spos[j], j) : nullptr;
      }
#pragma unroll
      for (int q = 0; q < GB; ++q) v[q] = ptr[q] ? __ldg(ptr[q]) : 0.0;
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int e = e0 + q * FNT;
        if (e < nT) T[(e % kpad) + (e / kpad) * LDT] = v[q];
      }
    }
    const int nM = nb * kpad;  // element e: row e % nb of column e / nb
    for (int e0 = tid; e0 < nM; e0 += GB * FNT) {
      const double* ptr[GB];
      double v[GB];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int e = e0 + q * FNT;
        const int r = e % nb, k = e / nb;
        ptr[q] = (e < nM && k < ni) ? entry_ptr(spos[ni + r], spos[k], k) : nullptr;
      }
#pragma unroll
      for (int q = 0; q < GB; ++q) v[q] = ptr[q] ? __ldg(ptr[q]) : 0.0;
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int e = e0 + q * FNT;
        if (e < nM) Mbi[(e % nb) + (e / nb) * LDB] = v[q];
      }
    }
  }
  __syncthreads();
  FCLK(1);
  // ---- LU of the ni interface rows with partial pivoting; columns [ni, total) ride along
  double pmin = DBL_MAX, pmax = 0.0;
  for (int k = 0; k < ni; ++k) {
    if (warp == 0) {
      // candidates: rows lane and lane + 32 in [k, ni)
      const double* ck = T + k * LDT;
      const int r0 = lane, r1 = lane + 32;
      const double a0 = (r0 >= k && r0 < ni) ? fabs(ck[r0]) : -1.0;
      const double a1 = (r1 >= k && r1 < ni) ? fabs(ck[r1]) : -1.0;
      // |a| as ordered bits (NaN sorts above inf: a NaN column still yields a flagged pivot)
      const bool take1 = a1 >= 0.0 && (a0 < 0.0 || __double_as_longlong(a1) > __double_as_longlong(a0));
      const double av = take1 ? a1 : a0;
      const int ar = take1 ? r1 : r0;
      const unsigned hi = av >= 0.0 || av != av ? (unsigned(__double2hiint(av)) | 0x80000000u) : 0u;
      const unsigned lo = unsigned(__double2loint(av));
      const unsigned whi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned wlo = __reduce_max_sync(0xffffffffu, hi == whi ? lo : 0u);
      const unsigned wrow = __reduce_min_sync(0xffffffffu, (hi == whi && lo == wlo) ? unsigned(ar) : 0xffffffffu);
      const int p = int(wrow);
      const double piv = ck[p];
      const double rinv = 1.0 / piv;
      const double akk = ck[k];
      // multipliers of the swapped column: row p holds the old row k
      if (r0 > k && r0 < ni) lvec[r0] = (r0 == p ? akk : ck[r0]) * rinv;
      if (r1 > k && r1 < ni) lvec[r1] = (r1 == p ? akk : ck[r1]) * rinv;
      if (lane == 0) {
        lvec[k] = 0.0;
        urinv[k] = rinv;
        s_piv = p;
        const double apv = fabs(piv);
        pmin = fmin(pmin, apv);
        pmax = (apv != apv) ? INFINITY : fmax(pmax, apv);
      }
    }
    __syncthreads();
    const int p = s_piv;
    if (tid >= k && tid < total) {
      double* cj = T + tid * LDT;
      const double a = cj[k], b = cj[p];
      cj[p] = a;
      cj[k] = b;
      if (tid > k) {
        const double u = -b;
        int i = (k + 1) & ~1;  // lvec[k] = 0 (and lvec[< k] = 0): an aligned pair may start at k
        // (rows up to kpad - 1 >= ni - 1 carry zero multipliers: whole batches of 4 pairs, loads
        // issued together -- a store between them would serialise on possible aliasing)
        for (; i + 8 <= kpad; i += 8) {
          double2 l[4], t[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) l[q] = f_lds128(lvec + i + 2 * q);
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] = f_lds128(cj + i + 2 * q);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            t[q].x = fma(l[q].x, u, t[q].x);
            t[q].y = fma(l[q].y, u, t[q].y);
            *reinterpret_cast<double2*>(cj + i + 2 * q) = t[q];
          }
        }
        for (; i < kpad; i += 2) {
          const double2 l = f_lds128(lvec + i);
          double2 t = f_lds128(cj + i);
          t.x = fma(l.x, u, t.x);
          t.y = fma(l.y, u, t.y);
          *reinterpret_cast<double2*>(cj + i) = t;
        }
      }
    }
    __syncthreads();
  }
  FCLK(2);
  // ---- X = U^{-1} Y, one boundary column per thread
  if (tid >= ni && tid < total) {
    double* cj = T + tid * LDT;
    for (int r = ni - 1; r >= 0; --r) {
      const double x = cj[r] * urinv[r];
      cj[r] = x;
      const double* ur = T + r * LDT;
      const double mx = -x;
      int i = 0;
      for (; i + 7 < r; i += 8) {
        double2 u[4], t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = f_lds128(ur + i + 2 * q);
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = f_lds128(cj + i + 2 * q);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          t[q].x = fma(u[q].x, mx, t[q].x);
          t[q].y = fma(u[q].y, mx, t[q].y);
          *reinterpret_cast<double2*>(cj + i + 2 * q) = t[q];
        }
      }
      for (; i + 1 < r; i += 2) {
        const double2 u = f_lds128(ur + i);
        double2 t = f_lds128(cj + i);
        t.x = fma(u.x, mx, t.x);
        t.y = fma(u.y, mx, t.y);
        *reinterpret_cast<double2*>(cj + i) = t;
      }
      if (i < r) cj[i] = fma(ur[i], mx, cj[i]);
    }
  }
  __syncthreads();
  FCLK(3);
  // ---- S = M_bb - M_bi X on the FP64 tensor cores, 32 x 32 blocks round-robin over the warps
  double* __restrict__ S = args.arena + nd.s_off;
  const long long lds = nd.ld;
  const int g = lane >> 2, tig = lane & 3;
  const int nbk = (nb + 31) >> 5;
  for (int blk = warp; blk < nbk * nbk; blk += FNT / 32) {
    const int r0 = (blk % nbk) * 32, c0 = (blk / nbk) * 32;
    double acc[2][4][4];
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      const double* ptr[2][2][2];
#pragma unroll
      for (int v2 = 0; v2 < 2; ++v2) {
        const int c = c0 + jn * 8 + 2 * tig + v2;
        const PosDev pc = spos[ni + min(c, nb - 1)];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + i * 16 + 2 * g + h;
            ptr[i][h][v2] = (r < nb && c < nb) ? entry_ptr(spos[ni + r], pc, ni + c) : nullptr;
          }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int v2 = 0; v2 < 2; ++v2) acc[i][jn][2 * h + v2] = ptr[i][h][v2] ? -__ldg(ptr[i][h][v2]) : 0.0;  // -M_bb
    }
    const double* ab = Mbi + r0 + 2 * g;
    const double* bb = T + (ni + c0 + g) * LDT + 2 * tig;
    for (int k8 = 0; k8 < kpad; k8 += 8) {
      double2 af[2][2], bf[4];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i][s] = f_lds128(ab + i * 16 + (k8 + 2 * tig + s) * LDB);
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) bf[jn] = f_lds128(bb + jn * 8 * LDT + k8);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
          mma_f64_m16n8k4(acc[i][jn], af[i][0].x, af[i][0].y, bf[jn].x);
          mma_f64_m16n8k4(acc[i][jn], af[i][1].x, af[i][1].y, bf[jn].y);
        }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int jn = 0; jn < 4; ++jn)
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
