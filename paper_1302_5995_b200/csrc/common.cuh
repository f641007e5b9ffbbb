// Shared device-side declarations for the B200 dense engine kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dtnb {

// Device copy of a plan node (plan.hpp:Node) — only what kernels read.
struct NodeDev {
  int kind;   // 0 micro, 1 merge, 2 root-LU workspace
  int nb, ni, total;
  int a, b;   // child node indices (merge)
  int ld;     // leading dimension of this node's S block
  int ldm;    // blocked: leading dimension of the assembled system
  long long s_off, m_off, pos_off, piv_off;
  long long rhs_off;  // body-load columns (nb x nloads, leading dimension rhs_ld)
  int rhs_ld;
  int ncols;          // blocked: columns of the assembled system (total + body-load columns)
  int defer;          // blocked Schur merge whose boundary columns skip the LU's row moves and rank-kb
                      // updates: Y = L^{-1} P M_ib is formed after the LU by blocked forward substitution
  // compressed engine (plan.hpp Node): structured merge / structured box
  int smerge;         // 1: M is the reduced interface system [[M_jj, Z], [W, 0]] (total = ni + sys_nb)
  int sys_nb;        // boundary columns of the blocked system (nb, or ra + rb for a structured merge)
  int j0, jn, ell;    // J edge range in the CCW boundary and the factor rank
  int ldq, ldf, ldg, ldr;
  long long q1_off, q2_off, rt_off, lk_off, om_off, y1_off, y2_off, lkg_off, rkg_off, tg_off;
};

constexpr int kProbes = 4;  // range-finder probe columns appended to every factor sketch

struct QrDesc {  // Householder QR of the first n columns of Y (m x (n + p), in place), the explicit Q
                 // (m x n), and the range-finder check of the p probe columns
  double* Y;
  double* Q;
  double* stat;     // [0] = #{|R_ii| > eps scale}, [1] = max over probes of |(I - Q Q^T) y| / scale
  const double* S;  // the box's S: scale = max_i |S_ii| sqrt(k / 3) (k = sketched columns, uniform[-1,1] probes)
  int ldy, ldq, m, n, p, lds, nbs, k;
};

struct RowGatherDesc {  // dst(i, c) = src(perm[i], c), i < rows, c < cols (perm: arena piv ints)
  const double* src;
  double* dst;
  long long perm_off;
  int lds, ldd, rows, cols;
};

struct PosDev {  // == plan.hpp PosEntry
  int src, partner, gid, dir;
};

struct GemmDesc {  // C(m x n) = beta*C + alpha*A(m x k)*B(k x n), column-major
  const double* A;
  const double* B;
  double* C;
  int m, n, k, lda, ldb, ldc;
};

struct SumDesc {  // dst(m x n, ldd) += sum_{s < slices} src + s * stride (m x n, lds each)
  double* dst;
  const double* src;
  long long stride;
  int ldd, lds, m, n, slices;
};

struct GemmDesc2 {  // C = A_cat B, A_cat = [A (row-major, first ka columns) | A2 (column-major)]
  const double* A;
  const double* A2;
  const double* B;
  double* C;
  int m, n, k, lda, lda2, ka, ka_valid, ldb, ldc;
};

struct TriDesc {  // inverses of the 128 x 128 diagonal blocks of U of an n x n LU
  const double* LU;
  double* out;
  int ld, n;
};

struct TrsmDesc {  // Y(bk x ncols) <- U^{-1} Y, U a bk x bk upper triangle (bk <= 128)
  const double* U;
  double* Y;
  int ldu, ldy, bk, ncols;
};

struct CopyDesc {
  const double* src;
  double* dst;
  int lds, ldd, m, n;
};

struct KernelArgs {
  const NodeDev* nodes;
  const PosDev* pos;
  const double* stencil;  // 5 x nu SoA: center, east, west, north, south
  long long nu;
  int side;               // n - 2
  double* arena;
  int* piv;
  double* pivstat;        // 2 per node: min |pivot|, max |pivot|
  int nl;                 // body-load columns carried through the build (0: none)
  const int* load_col;    // per unknown: its load column, or -1
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mma_f64_m16n8k4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; bytes < 16 zero-fills the remainder.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace dtnb
