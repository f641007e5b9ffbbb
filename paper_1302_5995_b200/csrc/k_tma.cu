// TMA-staged FP64 tensor-core GEMM for the large contractions of the merge (Schur
// complements S = M_bb - M_bi X, dense_nd.cpp:181; the structured updates S -= T R_k,
// accel_nd.cpp:551-621; the root inverse sweeps; the dense solve G X,
// solution_operator.cpp:36-52).
//
// 128 x 128 CTA tile, K in chunks of 16 through a 5-stage ring in shared memory. One
// elected thread issues the stage's tensor-map tile loads (cp.async.bulk.tensor.2d, SASS
// UTMALDG: 9 instructions per 32 KB stage) and the 8 math warps (64 x 32 warp tiles, DMMA
// m16n8k4) wait on the stage's "full" mbarrier and release it through an "empty" one: no
// per-thread global addresses, bounds predicates or copy instructions in the K loop. (A
// ninth, producer-only warp would cap the kernel at 168 registers -- warps are allocated in
// fours -- and spill the 128 accumulator registers.)
//
// Shared-memory layout (dense, hardware 128-byte swizzle, no padding):
//   A (column-major m x k, rows contiguous): 8 boxes of 16 rows x 16 k -> [box][k][16 rows],
//     one 128-byte line per k. The MMA's logical rows (g, g + 8) are mapped to the
//     ADJACENT physical rows (2g, 2g + 1), so both A fragments of a k step come from one
//     16-byte load; the accumulator rows are un-permuted in the epilogue.
//   B (column-major k x n, k contiguous): one box of 16 k x 128 columns -> [column][16 k].
//     The MMA's logical k index t of two consecutive k steps is mapped to the physical
//     k = 2t and 2t + 1 (A uses the same mapping), so one 16-byte load feeds both steps.
//   With the 128-byte swizzle (16-byte chunk index XOR line index mod 8) every warp-wide
//   fragment load touches each bank group exactly its minimum number of times.
// Rows / columns / k beyond the matrix are zero-filled by the TMA unit (tensor-map
// bounds), so ragged tiles need no predicates in the load path.
#include <cuda.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace dtnb {

constexpr int TBM = 128, TBN = 128, TBK = 16, TST = 5;
constexpr int TCONS = 256, TTHREADS = TCONS;  // 8 math warps; lane 0 of warp 0 is also the producer
constexpr int TLAG = 2;  // the producer refills the stage the warps left TLAG iterations ago (no stall on a laggard)
constexpr int TWM = 64, TWN = 32;
constexpr unsigned TSTAGE_A = TBM * TBK * 8, TSTAGE_B = TBN * TBK * 8;  // 16 KB each
constexpr unsigned TSTAGE = TSTAGE_A + TSTAGE_B;
constexpr size_t TMA_SMEM = size_t(TST) * TSTAGE + 1024;  // + alignment slack

__device__ __forceinline__ void tma_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// C = alpha A B + beta C over the descriptors' tiles (UPD: C -= A B with the C tile
// preloaded into the accumulators). tmaps[2 i], tmaps[2 i + 1]: the tensor maps of
// descriptor i's A and B (tma_encode_descs).
template <bool UPD>
__global__ void __launch_bounds__(TTHREADS, 1) gemm_tma_kernel(const GemmDesc* __restrict__ descs,
                                                               const CUtensorMap* __restrict__ tmaps, double alpha,
                                                               double beta) {
  extern __shared__ unsigned char tsm_raw[];
  __shared__ __align__(8) unsigned long long full[TST], empty[TST];
  const GemmDesc d = descs[blockIdx.y];
  const int m = d.m, n = d.n, k = d.k;
  const int tiles_m = (m + TBM - 1) / TBM, tiles_n = (n + TBN - 1) / TBN;
  if (int(blockIdx.x) >= tiles_m * tiles_n) return;
  const int row0 = (blockIdx.x % tiles_m) * TBM, col0 = (blockIdx.x / tiles_m) * TBN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned sbase = (smem_u32(tsm_raw) + 1023u) & ~1023u;  // 128-byte swizzle: 1024-byte aligned stages
  const int KT = (k + TBK - 1) / TBK;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TST; ++s) {
      tma_mbar_init(&full[s], 1);
      tma_mbar_init(&empty[s], TCONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // ---- producer duty (one thread): prologue fills TST - TLAG stages; at iteration kt the
  // stage consumed at kt - TLAG is refilled with chunk kt + TST - TLAG
  const CUtensorMap* tA = tmaps + 2 * blockIdx.y;
  const CUtensorMap* tB = tA + 1;
  unsigned char* gen = tsm_raw + (sbase - smem_u32(tsm_raw));
  auto produce = [&](int kl) {
    const int s = kl % TST;
    if (kl >= TST) tma_mbar_wait(&empty[s], unsigned((kl / TST) - 1) & 1u);
    tma_mbar_expect_tx(&full[s], TSTAGE);
    unsigned char* st = gen + size_t(s) * TSTAGE;
#pragma unroll
    for (int b = 0; b < TBM / 16; ++b) tma_load_2d(st + b * 2048, tA, row0 + 16 * b, kl * TBK, &full[s]);
    tma_load_2d(st + TSTAGE_A, tB, kl * TBK, col0, &full[s]);
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(tB) : "memory");
    for (int kl = 0; kl < TST - TLAG && kl < KT; ++kl) produce(kl);
  }
  // ---- consumers
  const int g = lane >> 2, tig = lane & 3;
  const int wm0 = (warp % (TBM / TWM)) * TWM, wn0 = (warp / (TBM / TWM)) * TWN;
  double acc[TWM / 16][TWN / 8][4];
#pragma unroll
  for (int i = 0; i < TWM / 16; ++i)
#pragma unroll
    for (int j = 0; j < TWN / 8; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        double x = 0.0;
        if constexpr (UPD) {  // acc = -C, result C - A B = -(acc + A B)
          const int r = row0 + wm0 + i * 16 + 2 * g + (v >> 1);
          const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
          if (r < m && c < n) x = -d.C[r + (long long)c * d.ldc];
        }
        acc[i][j][v] = x;
      }
  // per-thread fragment addresses within a stage (the swizzle XOR is folded in)
  //   A: box (wm0 / 16 + i), line kp = 8 p + 2 tig + s (s = k step of the pair), chunk g
  //   B: line (wn0 + 8 j + g) (line mod 8 = g), chunk 4 p + tig
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % TST;
    if (tid == 0 && kt + TST - TLAG < KT) produce(kt + TST - TLAG);
    tma_mbar_wait(&full[s], unsigned(kt / TST) & 1u);
    const unsigned sa = sbase + unsigned(s) * TSTAGE + unsigned(wm0 / 16) * 2048u;
    const unsigned sb = sbase + unsigned(s) * TSTAGE + TSTAGE_A + unsigned(wn0 + g) * 128u;
#pragma unroll
    for (int p = 0; p < TBK / 8; ++p) {
      double2 af[TWM / 16][2], bf[TWN / 8];
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const int kp = 8 * p + 2 * tig + st;
        const unsigned off = unsigned(kp) * 128u + (unsigned(g ^ (kp & 7)) << 4);
#pragma unroll
        for (int i = 0; i < TWM / 16; ++i) af[i][st] = lds128(sa + unsigned(i) * 2048u + off);
      }
#pragma unroll
      for (int j = 0; j < TWN / 8; ++j) bf[j] = lds128(sb + unsigned(j) * 1024u + (unsigned((4 * p + tig) ^ g) << 4));
#pragma unroll
      for (int i = 0; i < TWM / 16; ++i)
#pragma unroll
        for (int j = 0; j < TWN / 8; ++j) {
          mma_f64_m16n8k4(acc[i][j], af[i][0].x, af[i][0].y, bf[j].x);
          mma_f64_m16n8k4(acc[i][j], af[i][1].x, af[i][1].y, bf[j].y);
        }
    }
    __syncwarp();
    if (lane == 0) tma_mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int i = 0; i < TWM / 16; ++i)
#pragma unroll
    for (int j = 0; j < TWN / 8; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = row0 + wm0 + i * 16 + 2 * g + (v >> 1);
        const int c = col0 + wn0 + j * 8 + 2 * tig + (v & 1);
        if (r < m && c < n) {
          double* pc = d.C + r + (long long)c * d.ldc;
          if constexpr (UPD) *pc = -acc[i][j][v];
          else *pc = beta == 0.0 ? alpha * acc[i][j][v] : fma(alpha, acc[i][j][v], beta * *pc);
        }
      }
}

// ---- host side: tensor maps for descriptor arrays --------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn tma_encoder() {
  static const EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// DTN_GEMM_TMA=0 keeps the cp.async large-tile kernel (A/B switch)
bool gemm_tma_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("DTN_GEMM_TMA");
    return !(e && e[0] == '0') && tma_encoder() != nullptr;
  }();
  return v;
}

static bool tma_encode_2d(CUtensorMap* out, const double* base, uint64_t inner, uint64_t outer, uint64_t ld,
                          uint32_t box_inner, uint32_t box_outer) {
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (ld & 1u) || inner == 0 || outer == 0) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 8};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  return tma_encoder()(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor maps (A then B) of count descriptors whose pointers are DEVICE addresses; ok[i] = 0
// where a descriptor cannot be loaded by TMA (unaligned base, odd leading dimension, or a
// contraction too short to be worth it) -- launches containing such a descriptor keep the
// cp.async kernels. Returns false if the driver has no tensor-map encoder.
bool tma_encode_descs(const GemmDesc* h, size_t count, std::vector<CUtensorMap>& maps, std::vector<char>& ok) {
  maps.assign(2 * count, CUtensorMap{});
  ok.assign(count, 0);
  if (!gemm_tma_enabled()) return false;
  for (size_t i = 0; i < count; ++i) {
    const GemmDesc& d = h[i];
    if (d.m <= 0 || d.n <= 0 || d.k < 64 || !d.A || !d.B) continue;
    if (int64_t(d.m) * d.n < 128 * 128) continue;
    ok[i] = tma_encode_2d(&maps[2 * i], d.A, uint64_t(d.m), uint64_t(d.k), uint64_t(d.lda), 16, TBK) &&
            tma_encode_2d(&maps[2 * i + 1], d.B, uint64_t(d.k), uint64_t(d.n), uint64_t(d.ldb), TBK, TBN);
  }
  return true;
}

cudaError_t gemm_tma_init() {
  cudaError_t e = cudaFuncSetAttribute(gemm_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TMA_SMEM));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(gemm_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TMA_SMEM));
}

// max_tiles: an upper bound of the 128 x 128 tile count of the launch's largest descriptor
cudaError_t launch_gemm_tma(const GemmDesc* d_descs, const void* d_tmaps, int count, int max_tiles, double alpha,
                            double beta, cudaStream_t st) {
  if (count <= 0 || max_tiles <= 0) return cudaSuccess;
  dim3 grid(max_tiles, count);
  const CUtensorMap* tm = static_cast<const CUtensorMap*>(d_tmaps);
  if (alpha == -1.0 && beta == 1.0) gemm_tma_kernel<true><<<grid, TTHREADS, TMA_SMEM, st>>>(d_descs, tm, alpha, beta);
  else gemm_tma_kernel<false><<<grid, TTHREADS, TMA_SMEM, st>>>(d_descs, tm, alpha, beta);
  return cudaGetLastError();
}

}  // namespace dtnb

// ---- tensor-map sets for the engine's descriptor arrays (engine.cu holds them opaquely)
namespace dtnb {

// Device array of 2 * count tensor maps for a host copy of a descriptor array (device
// pointers); ok[i] as tma_encode_descs. nullptr when nothing can use TMA.
void* tma_build_set(const GemmDesc* h, size_t count, std::vector<char>& ok) {
  std::vector<CUtensorMap> maps;
  if (count == 0 || !tma_encode_descs(h, count, maps, ok)) return nullptr;
  bool any = false;
  for (char c : ok) any = any || c;
  if (!any) return nullptr;
  void* d = nullptr;
  if (cudaMalloc(&d, maps.size() * sizeof(CUtensorMap)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

// the maps of descriptors [off, off + cnt), or nullptr unless every one of them has maps
const void* tma_slice(const void* set, const std::vector<char>& ok, size_t off, size_t cnt) {
  if (!set || off + cnt > ok.size()) return nullptr;
  for (size_t i = off; i < off + cnt; ++i)
    if (!ok[i]) return nullptr;
  return static_cast<const CUtensorMap*>(set) + 2 * off;
}

// one descriptor's two maps into a caller buffer of 256 bytes (per-call descriptors: the solve)
bool tma_encode_one(const GemmDesc& d, void* out256) {
  std::vector<CUtensorMap> maps;
  std::vector<char> ok;
  if (!tma_encode_descs(&d, 1, maps, ok) || !ok[0]) return false;
  std::memcpy(out256, maps.data(), 2 * sizeof(CUtensorMap));
  return true;
}

// Launch threshold in 128 x 64 tiles of the launch (measured, tools/probe/tma_probe.cu: the
// TMA kernel matches the cp.async kernels at 1916 x 2044 x 128 and wins above)
int gemm_tma_min_tiles() {
  static const int v = [] {
    const char* t = std::getenv("DTN_GEMM_TMA_TILES");
    return t ? std::atoi(t) : 480;
  }();
  return v;
}

}  // namespace dtnb
