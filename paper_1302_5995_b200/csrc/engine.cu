// Host orchestration of the B200 dense engine and the C ABI (include/dtn_gpu.h).
//
// One build = one CUDA-graph launch of: per wave, the batched one-CTA
// eliminations (micro boxes and small merges, k_small.cu) and the blocked
// merges (gather + panel/rowpanel/trailing per kb pivots, k_blocked.cu,
// k_gemm.cu); then the root inverse G = S^{-1} (blocked LU of S with the same
// kernels, then forward/backward blocked triangular sweeps on P*I). The plan
// (tree, DAG, position tables, arena layout, graph) is cached per context.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/dtn_gpu.h"
#include "common.cuh"
#include "plan.hpp"
#include "hbs.hpp"
#include "nccl_dl.hpp"

namespace dtnb {
cudaError_t launch_small_elim(const KernelArgs&, const int*, int, int, bool, cudaStream_t);
cudaError_t launch_gather(const KernelArgs&, const int*, int, int, cudaStream_t);
cudaError_t launch_panel(const KernelArgs&, const int*, int, int, int, int, cudaStream_t, bool);
bool panel_is_tall(int max_rows);
int panel_tall_max_rows(int count);
cudaError_t launch_rowpanel(const KernelArgs&, const int*, int, int, int, int, int, bool, cudaStream_t, bool);
cudaError_t launch_trailing_update(const KernelArgs&, const int*, int, int, int, int, int, int, cudaStream_t, int);
cudaError_t launch_tri_inv_u_batched(const void*, int, int, cudaStream_t);
cudaError_t launch_copy2d_batched(const void*, int, cudaStream_t);
cudaError_t launch_trsm_upper_batched(const void*, int, int, cudaStream_t);
cudaError_t launch_trsm_batched(const void*, int, int, int, bool, cudaStream_t);
cudaError_t launch_block_identity(double*, int, cudaStream_t);
unsigned panel_fallbacks_read_reset();
unsigned small_fallbacks_read_reset();
cudaError_t launch_ring_dtn(const double*, int, const int*, const double*, int, double, double*, long long, cudaStream_t);
cudaError_t launch_trsm_upper_ref(const void*, int, int, cudaStream_t);
cudaError_t launch_gemm_desc(const GemmDesc*, int, int, int, double, double, cudaStream_t, bool, bool allow_big = true);
cudaError_t launch_pivot_screen(const double*, const int*, int, int, int*, cudaStream_t);
cudaError_t launch_row_gather(const RowGatherDesc*, int, const int*, cudaStream_t);
cudaError_t launch_skinny_gemm(const double*, int, const double*, int, double*, int, int, int, int, double*,
                               cudaStream_t);
size_t skinny_work_doubles(int, int, int);
cudaError_t launch_perm_identity(const int*, int, int*, double*, int, cudaStream_t);
cudaError_t launch_trsm_rows(const double*, int, double*, int, int, int, int, bool, cudaStream_t);
cudaError_t launch_norm1(const double*, int, int, int, unsigned long long*, cudaStream_t);
cudaError_t launch_copy2d(const double*, int, double*, int, int, int, cudaStream_t);
cudaError_t gemm_init();
cudaError_t gemm_tma_init();
cudaError_t fused_init();
void fused_clocks_read(long long*);
bool fused_merge_fits(int, int, int);
cudaError_t launch_fused_merge(const KernelArgs&, const int*, int, int, int, int, cudaStream_t);
void* tma_build_set(const GemmDesc*, size_t, std::vector<char>&);
const void* tma_slice(const void*, const std::vector<char>&, size_t, size_t);
bool tma_encode_one(const GemmDesc&, void*);
int gemm_tma_min_tiles();
cudaError_t launch_gemm_tma(const GemmDesc*, const void*, int, int, double, double, cudaStream_t);
cudaError_t misc_init();
cudaError_t launch_tri_inv_blocks(const double*, int, int, double*, cudaStream_t);
cudaError_t launch_set_identity(double*, int, int, cudaStream_t);
cudaError_t launch_permute_columns(const double*, int, const int*, int, double*, int, cudaStream_t);
cudaError_t launch_perm_only(const int*, int, int*, cudaStream_t);
cudaError_t blocked_init();
cudaError_t hbs_kernels_init();
cudaError_t struct_init();
cudaError_t launch_perm_identity_cols(const int*, int, int, int, double*, int, cudaStream_t);
cudaError_t launch_sgather_red(const KernelArgs&, const int*, int, int, cudaStream_t);
cudaError_t launch_kk_gather(const KernelArgs&, const int*, int, int, cudaStream_t);
cudaError_t launch_factor_gather(const KernelArgs&, const int*, int, long long, cudaStream_t);
cudaError_t launch_omega(const KernelArgs&, const int*, int, long long, cudaStream_t);
cudaError_t launch_sum_partials(const SumDesc*, int, long long, cudaStream_t);
cudaError_t launch_hqr(const QrDesc*, int, int, int, const double*, cudaStream_t, bool = false);
cudaError_t launch_gemm_desc2(const GemmDesc2*, int, int, bool, cudaStream_t);
int gemm_tiles(int, int);
extern std::atomic<unsigned long long> g_hbs_launches;
}  // namespace dtnb

using namespace dtnb;

namespace {

struct CudaFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Singular : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw CudaFail(std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

constexpr int kSmallMax = 160;
constexpr int kDefaultMicro = 16;  // measured best on configs 1-2 (tools/sweep.py)

// Panel width; the register-resident cluster panel spans up to 16 CTAs x 512 rows, the
// tall panel (global-memory pivot exchange) up to 512 rows per SM.
int panel_kb(int rows, int count = 1) {
  if (rows > 16 * 512 && rows > panel_tall_max_rows(count))
    throw std::invalid_argument("dense merge system too large for the tall panel (" + std::to_string(rows) +
                                " rows, " + std::to_string(count) + " systems)");
  return 32;
}

struct WaveLaunch {
  int micro_off = 0, micro_cnt = 0, micro_max = 0;
  int small_off = 0, small_cnt = 0, small_max = 0;
  int blk_off = 0, blk_cnt = 0, blk_max_total = 0, blk_max_ni = 0, blk_max_nb = 0, kb = 32;
  int level = -1;  // reference level of its tree merges, -1 for in-leaf waves
  double flops = 0.0;
  // Schur-form back substitution X = U^{-1} Y and S -= M_bi X (descriptor ranges)
  int tri_off = 0, tri_blocks = 0;                 // TriDesc range (one per blocked merge)
  std::vector<int> bs_off, bs_cnt;                 // per back-substitution step: GemmDesc pairs / CopyDesc
  std::vector<int> bs_toff, bs_soff, bs_tiles1, bs_tiles2, bs_k, bs_cols;  // launch geometry per step
  std::vector<double> bs_flops;
  int copy_base = 0;                               // first CopyDesc of this wave
  // deferred boundary columns (NodeDev::defer): copy out, row gather by the LU's
  // permutation, then Y = L^{-1} (P M_ib) by 128-row blocks (unit-lower substitution + GEMM)
  int fw_copy_off = 0, fw_cnt = 0, fw_gather_off = 0, fw_max_cols = 0;
  std::vector<int> fw_toff, fw_goff, fw_n, fw_tiles, fw_k, fw_cols;
  std::vector<double> fw_flops;
  int fin_off = 0, fin_tiles = 0, fin_k = 0, fin_cnt = 0;  // final GEMM S -= M_bi X (descriptors)
  std::vector<int> gather_nodes;                   // column-sharded merges: ncclAllGather after the wave
  bool fin_aligned = true;
  double fin_flops = 0.0;
  // compressed engine: dense blocked merges (gather) vs structured merges (reduced system)
  int gd_off = 0, gd_cnt = 0, gd_max_total = 0;
  int sm_off = 0, sm_cnt = 0, sm_max_total = 0, sm_max_nb = 0;
  long long sm_max_elems = 0;
  int sm_copy = 0;                                  // CopyDesc: C -> aligned buffer
  int sm_t = 0, sm_t_tiles = 0, sm_t_k = 0;         // GemmDesc: T = -L_k C
  int sm_u = 0, sm_u_tiles = 0, sm_u_k = 0;         // GemmDesc: S -= T R_k
  double sm_flops = 0.0;
  int cp_off = 0, cp_cnt = 0;
  long long cp_max_elems = 0;
  int cp_y1 = 0, cp_y1_n = 0, cp_y1_tiles = 0, cp_y1_k = 0;  // GemmDesc:  Y1 = S[J, :] Omega (K-slices)
  int cp_y2 = 0, cp_y2_n = 0, cp_y2_tiles = 0;                // GemmDesc2: Y2 = S[:, J]^T Omega (K-slices)
  int cp_sum = 0, cp_sum_n = 0;                               // SumDesc: the slices into Y1 / Y2
  long long cp_sum_elems = 0;
  int cp_qr = 0, cp_qr_m = 0, cp_qr_n = 0;          // QrDesc x 2 cp_cnt
  int cp_rt = 0, cp_rt_tiles = 0;                   // GemmDesc2: R_jk^T = S[J, :]^T Q1
  int cp_lk = 0, cp_lk_tiles = 0, cp_lk_k = 0;      // GemmDesc:  L_kj = S[:, J] Q2
  bool cp_lk_aligned = true;
  double cp_flops = 0.0;
};

template <class T>
T* dalloc(size_t count) {
  T* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return p;
}

// Tensor maps of a descriptor array (k_tma.cu): launches whose descriptors all have maps and
// that are large enough run the TMA-staged kernel, the others the cp.async kernels.
struct TmaSet {
  void* d = nullptr;
  std::vector<char> ok;
  void build(const std::vector<GemmDesc>& h) {
    if (d) cudaFree(d);
    d = tma_build_set(h.data(), h.size(), ok);
  }
  const void* slice(size_t off, size_t cnt) const { return tma_slice(d, ok, off, cnt); }
  ~TmaSet() {
    if (d) cudaFree(d);
  }
};

cudaError_t gemm_go(const GemmDesc* base, const TmaSet& tm, size_t off, int cnt, int max_tiles, int kmax, double alpha,
                    double beta, cudaStream_t st, bool aligned) {
  const void* maps =
      (kmax >= 64 && int64_t(max_tiles) * cnt >= gemm_tma_min_tiles()) ? tm.slice(off, size_t(cnt)) : nullptr;
  if (maps) return launch_gemm_tma(base + off, maps, cnt, max_tiles, alpha, beta, st);
  return launch_gemm_desc(base + off, cnt, max_tiles, kmax, alpha, beta, st, aligned);
}

struct PlanDev {
  TmaSet tm_bs, tm_sg, tm_rg, tm_inv, tm_fw;
  Plan P;
  bool busy = false;
  int device = 0;
  std::vector<NodeDev> h_nodes;
  NodeDev* d_nodes = nullptr;
  PosDev* d_pos = nullptr;
  double* d_arena = nullptr;
  int* d_piv = nullptr;
  double* d_pivstat = nullptr;
  int* d_lists = nullptr;
  std::vector<int> h_lists;
  double* d_stencil = nullptr;
  int64_t nu = 0;
  std::vector<WaveLaunch> wl;
  int root_list_off = 0, root_lu_node = 0;
  int nb = 0;           // root boundary size
  double* d_S = nullptr;  // compact root S (ld = lds)
  int lds = 0;
  double* d_G = nullptr;
  int ldg = 0;
  int64_t lu_off = 0;
  int ldlu = 0, root_kb = 32;
  int* d_perm = nullptr;
  unsigned long long* d_norm = nullptr;
  GemmDesc* d_inv_descs = nullptr;
  std::vector<GemmDesc> h_inv_descs;
  std::vector<GemmDesc> h_bs_gemm;  // arena offsets until relocated
  std::vector<CopyDesc> h_bs_copy;
  std::vector<TriDesc> h_tri;
  std::vector<TrsmDesc> h_trs;
  std::vector<CopyDesc> h_fw_copy;
  std::vector<RowGatherDesc> h_fw_gather;
  std::vector<TrsmDesc> h_fw_trs;
  std::vector<GemmDesc> h_fw_gemm;
  CopyDesc* d_fw_copy = nullptr;
  RowGatherDesc* d_fw_gather = nullptr;
  TrsmDesc* d_fw_trs = nullptr;
  GemmDesc* d_fw_gemm = nullptr;
  int64_t gtmp_off = 0, gtmp_doubles = 0;
  int subst_base = 0;
  TrsmDesc* d_trs = nullptr;
  GemmDesc* d_bs_gemm = nullptr;  // back-substitution / final GEMM descriptors (all waves)
  CopyDesc* d_bs_copy = nullptr;
  TriDesc* d_tri = nullptr;
  double* d_W = nullptr;     // U^{-1} L^{-1} before the column permutation
  double* d_LUp = nullptr;   // L_ik Linv_kk (below) and U_ik Uinv_kk (above the diagonal blocks)
  double* d_UI = nullptr;    // U^{-1} before its deferred diagonal-block solves, then U^{-1} (d_UI2)
  double* d_UI2 = nullptr;
  int inv_ui = 0;            // descriptor ranges: U^{-1} sweep, U^{-1} block solves, final product
  int* d_load_col = nullptr;  // body loads: per unknown, its load column or -1
  double* d_F = nullptr;      // body map F = G * rhs_root (nb x nloads, leading dimension ldf)
  int ldf = 0;
  GemmDesc h_F_desc{};
  GemmDesc* d_F_desc = nullptr;
  int64_t rhs_root_off = 0;
  int rhs_root_ld = 0;
  int inv_pre = 0;           // pre-product descriptors at the front of h_inv_descs
  std::vector<TrsmDesc> h_root_trs;
  TrsmDesc* d_root_trs = nullptr;
  double* d_tinv = nullptr;  // inverses of the 128 x 128 diagonal blocks of L and U
  double* h_pivstat = nullptr;  // pinned
  int* d_chk = nullptr;         // per node: 1 checked for singular pivots, 2 only when G is built
  int* d_bad = nullptr;         // lowest failing node id (INT_MAX: none)
  int* h_bad = nullptr;         // pinned
  unsigned long long* h_norm = nullptr;
  std::vector<cudaEvent_t> ev_wave;
  cudaEvent_t ev_start = nullptr, ev_root = nullptr, ev_end = nullptr;
  cudaEvent_t ev_rp = nullptr, ev_rest = nullptr;  // look-ahead dependencies
  cudaEvent_t ev_rest2[2] = {nullptr, nullptr};       // fused look-ahead: side-stream step parity
  cudaEvent_t ev_S = nullptr;                           // root S complete (external node in the graph)
  cudaEvent_t ev_inv_fork = nullptr, ev_inv_join = nullptr;  // root inverse: U^{-1} on the side stream
  cudaStream_t copy = nullptr;                          // S export overlapping the root inverse
  cudaStream_t side = nullptr;                      // low-priority stream for trailing updates
  cudaGraphExec_t gexec = nullptr;
  int graph_want_G = -1;
  int launches = 0;
  void* comm = nullptr;  // ncclComm_t of a collective top build (the context's)
  // collective top build: G by column chunks, G[:, c0:c1] = U^{-1} L^{-1} P[:, c0:c1]
  // (forward / backward block substitution on the root LU, this rank's chunk)
  int root_cw = 0;
  std::vector<std::pair<int, int>> root_chunks;
  std::vector<GemmDesc> h_rg;  // per block step: forward updates, then backward updates
  std::vector<TrsmDesc> h_rt;  // per block step: forward (unit lower), then backward (upper)
  std::vector<int> rg_off, rg_cnt, rt_off, rt_cnt;  // [0, nblk) forward steps, [nblk, 2 nblk) backward
  GemmDesc* d_rg = nullptr;
  TrsmDesc* d_rt = nullptr;
  // compressed engine descriptors (arena offsets relocated at upload) and statistics
  std::vector<CopyDesc> h_sm_copy;
  std::vector<GemmDesc> h_sg;
  std::vector<GemmDesc2> h_sg2;
  std::vector<SumDesc> h_sum;
  SumDesc* d_sum = nullptr;
  std::vector<QrDesc> h_qr;
  CopyDesc* d_sm_copy = nullptr;
  GemmDesc* d_sg = nullptr;
  GemmDesc2* d_sg2 = nullptr;
  QrDesc* d_qr = nullptr;
  double* d_eps = nullptr;     // sketch rank threshold (written before every launch)
  double* d_qstat = nullptr;   // per QR: numerical rank, tail (QrDesc::stat)
  double* h_qstat = nullptr;   // pinned
  std::vector<int> qr_node;    // node of each QR

  ~PlanDev() {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (auto e : ev_wave) cudaEventDestroy(e);
    for (auto e : {ev_start, ev_root, ev_end, ev_rp, ev_rest, ev_rest2[0], ev_rest2[1], ev_S, ev_inv_fork, ev_inv_join})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (copy) cudaStreamDestroy(copy);
    for (void* p : std::initializer_list<void*>{d_nodes, d_pos, d_arena, d_piv, d_pivstat, d_lists, d_stencil, d_S, d_G,
                                                d_perm, d_norm, d_inv_descs, d_W, d_LUp, d_UI, d_UI2, d_tinv, d_root_trs, d_load_col, d_F, d_F_desc, d_bs_gemm,
                                                d_bs_copy, d_tri, d_trs, d_chk, d_bad, d_fw_copy, d_fw_gather,
                                                d_fw_trs, d_fw_gemm, d_sm_copy, d_sg, d_sg2, d_sum, d_qr, d_eps, d_qstat, d_rg, d_rt})
      if (p) cudaFree(p);
    if (h_qstat) cudaFreeHost(h_qstat);
    if (h_pivstat) cudaFreeHost(h_pivstat);
    if (h_bad) cudaFreeHost(h_bad);
    if (h_norm) cudaFreeHost(h_norm);
  }

  KernelArgs args() const {
    return KernelArgs{d_nodes, d_pos,    d_stencil, (long long)nu, P.n - 2, d_arena,
                      d_piv,   d_pivstat, P.key.nloads,  d_load_col};
  }
};

double defer_min_work();

std::unique_ptr<PlanDev> make_plandev(const PlanKey& key, int device) {
  auto D = std::make_unique<PlanDev>();
  D->device = device;
  D->P = make_plan(key);
  Plan& P = D->P;
  D->nu = int64_t(P.n - 2) * (P.n - 2);
  const Node& root = P.nodes[P.root];
  D->nb = root.nb;
  const int nb = D->nb;
  // nodes (+ the root-LU pseudo node)
  D->h_nodes.resize(P.nodes.size() + 1);
  for (size_t i = 0; i < P.nodes.size(); ++i) {
    const Node& s = P.nodes[i];
    NodeDev& d = D->h_nodes[i];
    d.kind = int(s.kind);
    d.nb = s.nb;
    d.ni = s.ni;
    d.total = s.total;
    d.a = s.a;
    d.b = s.b;
    d.ld = s.ld;
    d.ldm = s.ldm;
    d.s_off = s.s_off;
    d.m_off = s.m_off;
    d.pos_off = s.pos_off;
    d.piv_off = s.piv_off;
    d.rhs_off = s.rhs_off;
    d.rhs_ld = s.rhs_ld;
    d.ncols = s.total + (s.blocked ? P.key.nloads : 0);
    d.defer = 0;  // decided per wave below
    d.smerge = s.smerge ? 1 : 0;
    d.sys_nb = s.sys_nb;
    d.j0 = s.j0;
    d.jn = s.jn;
    d.ell = s.ell;
    d.ldq = s.ldq;
    d.ldf = s.ldf;
    d.ldg = s.ldg;
    d.ldr = s.ldr;
    d.q1_off = s.q1_off;
    d.q2_off = s.q2_off;
    d.rt_off = s.rt_off;
    d.lk_off = s.lk_off;
    d.om_off = s.om_off;
    d.y1_off = s.y1_off;
    d.y2_off = s.y2_off;
    d.lkg_off = s.lkg_off;
    d.rkg_off = s.rkg_off;
    d.tg_off = s.tg_off;
  }
  D->ldlu = int(align_up(nb, 8));
  D->lu_off = align_up(P.arena_doubles, 32);
  D->root_lu_node = int(P.nodes.size());
  {
    NodeDev& r = D->h_nodes.back();
    std::memset(&r, 0, sizeof(r));
    r.kind = 2;
    r.nb = 0;
    r.ni = nb;
    r.total = nb;
    r.a = r.b = -1;
    r.ldm = D->ldlu;
    r.ld = D->ldlu;
    r.m_off = D->lu_off;
    r.s_off = D->lu_off;
    r.ncols = nb;
    r.piv_off = P.piv_ints;
  }
  D->root_kb = 32;  // (the root LU's row limit is checked when G is requested)
  // launch lists
  std::vector<int> lists;
  D->wl.resize(P.waves.size());
  for (size_t w = 0; w < P.waves.size(); ++w) {
    const Wave& wv = P.waves[w];
    WaveLaunch& L = D->wl[w];
    L.micro_off = int(lists.size());
    L.micro_cnt = int(wv.micro.size());
    for (int id : wv.micro) {
      lists.push_back(id);
      L.micro_max = std::max(L.micro_max, P.nodes[id].total + P.key.nloads);
    }
    L.small_off = int(lists.size());
    L.small_cnt = int(wv.small.size());
    for (int id : wv.small) {
      lists.push_back(id);
      L.small_max = std::max(L.small_max, P.nodes[id].total + P.key.nloads);
    }
    L.blk_off = int(lists.size());
    L.blk_cnt = int(wv.blocked.size());
    for (int id : wv.blocked) {
      lists.push_back(id);
      const Node& nd = P.nodes[id];
      L.blk_max_total = std::max(L.blk_max_total, nd.total);
      L.blk_max_ni = std::max(L.blk_max_ni, nd.ni);
      L.blk_max_nb = std::max(L.blk_max_nb, nd.nb);
    }
    if (L.blk_cnt) L.kb = panel_kb(L.blk_max_ni, L.blk_cnt);
    L.gd_off = int(lists.size());
    for (int id : wv.blocked)
      if (!P.nodes[id].smerge) {
        lists.push_back(id);
        ++L.gd_cnt;
        L.gd_max_total = std::max(L.gd_max_total, P.nodes[id].total);
      }
    L.sm_off = int(lists.size());
    for (int id : wv.smerge) {
      const Node& nd = P.nodes[id];
      lists.push_back(id);
      ++L.sm_cnt;
      L.sm_max_total = std::max(L.sm_max_total, nd.total);
      L.sm_max_nb = std::max(L.sm_max_nb, nd.nb);
      L.sm_max_elems = std::max<long long>(L.sm_max_elems, (long long)nd.nb * nd.sys_nb);
    }
    L.cp_off = int(lists.size());
    for (int id : wv.compress) {
      const Node& nd = P.nodes[id];
      lists.push_back(id);
      ++L.cp_cnt;
      L.cp_max_elems = std::max<long long>(L.cp_max_elems, (long long)nd.nb * (nd.ell + kProbes));
    }
    for (int id : wv.small) {
      const Node& nd = P.nodes[id];
      if (nd.label_level >= 0) L.level = L.level < 0 ? nd.label_level : std::min(L.level, nd.label_level);
    }
    for (int id : wv.blocked) {
      const Node& nd = P.nodes[id];
      if (nd.label_level >= 0) L.level = L.level < 0 ? nd.label_level : std::min(L.level, nd.label_level);
    }
    for (int id : wv.small) L.flops += merge_flop_count(P.nodes[id].ni, P.nodes[id].nb);
    for (int id : wv.blocked) L.flops += merge_flop_count(P.nodes[id].ni, P.nodes[id].nb);
    for (int id : wv.micro) L.flops += merge_flop_count(P.nodes[id].ni, P.nodes[id].nb);
  }
  // Schur-form descriptors: X = U^{-1} Y by 128-row blocks from the bottom
  // (T = Uinv_k Y_k; Y_top -= U_top,k T; Y_k = T), then S -= M_bi X. Every
  // descriptor covers one column segment [c0, c1) of a node's boundary columns:
  // the whole range, or (collective top build, Node::colshard) this rank's chunk
  // -- or every rank's chunk in turn when the split is checked on one device.
  {
    std::vector<GemmDesc> gd;
    std::vector<CopyDesc> cd;
    std::vector<TriDesc> td;
    std::vector<TrsmDesc> trs;
    std::vector<GemmDesc> gs;  // substitution variant's updates (appended after gd)
    std::vector<CopyDesc> fwc;
    std::vector<RowGatherDesc> fwg;
    std::vector<TrsmDesc> fwt;
    std::vector<GemmDesc> fwm;
    int64_t gtmp_need = 0;
    // the deferred columns' staging area sits after the root-LU region of the arena
    D->gtmp_off = align_up(D->lu_off + int64_t(D->ldlu) * nb, 32);
    auto segs = [&](const Node& nd) {
      std::vector<std::pair<int, int>> out;
      const int ncy = nd.sys_nb + P.key.nloads;
      if (!nd.colshard) {
        out.push_back({0, ncy});
        return out;
      }
      for (int r = 0; r < P.key.world; ++r) {
        if (P.key.wrank >= 0 && r != P.key.wrank) continue;
        const int c0 = r * nd.cw, c1 = std::min(ncy, c0 + nd.cw);
        if (c1 > c0) out.push_back({c0, c1});
      }
      return out;
    };
    for (size_t w = 0; w < P.waves.size(); ++w) {
      WaveLaunch& L = D->wl[w];
      const Wave& wv = P.waves[w];
      if (wv.blocked.empty()) continue;
      L.tri_off = int(td.size());
      int maxblk = 0;
      for (int id : wv.blocked) {
        const Node& nd = P.nodes[id];
        td.push_back(TriDesc{reinterpret_cast<const double*>(nd.m_off), reinterpret_cast<double*>(nd.uinv_off), nd.ldm,
                             nd.ni});
        maxblk = std::max(maxblk, (nd.ni + 127) / 128);
      }
      L.tri_blocks = maxblk;
      // deferred boundary columns: M_ib -> temp (ni x ncy), gathered back by perm,
      // then forward substitution by 128-row blocks (top down). Decided per wave by
      // the boundary-column work of its rank-32 updates, sum of ni (ncols - ni);
      // always for column-sharded merges (their LU must not touch the boundary columns)
      {
        double work = 0.0;
        for (int id : wv.blocked) work += double(P.nodes[id].ni) * double(D->h_nodes[id].ncols - P.nodes[id].ni);
        if (work >= defer_min_work())
          for (int id : wv.blocked) D->h_nodes[id].defer = P.nodes[id].ni >= 256 ? 1 : 0;
        for (int id : wv.blocked)
          if (P.nodes[id].colshard) D->h_nodes[id].defer = 1;
      }
      {
        int64_t toff = D->gtmp_off;
        L.fw_copy_off = int(fwc.size());
        L.fw_gather_off = int(fwg.size());
        int fmax = 0;
        for (int id : wv.blocked) {
          const Node& nd = P.nodes[id];
          if (!D->h_nodes[id].defer) continue;
          const int64_t M = nd.m_off, ldm = nd.ldm;
          const int ldt = int(align_up(nd.ni, 2));
          for (auto [c0, c1] : segs(nd)) {
            const int ncy = c1 - c0;
            const int64_t Yc = M + (int64_t(nd.ni) + c0) * ldm;
            fwc.push_back(CopyDesc{reinterpret_cast<const double*>(Yc), reinterpret_cast<double*>(toff), int(ldm), ldt,
                                   nd.ni, ncy});
            fwg.push_back(RowGatherDesc{reinterpret_cast<const double*>(toff), reinterpret_cast<double*>(Yc),
                                        nd.piv_off, ldt, int(ldm), nd.ni, ncy});
            toff += int64_t(ldt) * ncy;
            ++L.fw_cnt;
            L.fw_max_cols = std::max(L.fw_max_cols, ncy);
          }
          fmax = std::max(fmax, (nd.ni + 127) / 128);
        }
        gtmp_need = std::max(gtmp_need, toff - D->gtmp_off);
        for (int t = 0; t < fmax; ++t) {
          int cnt = 0, tiles = 0, kk = 0, mc = 0;
          double fl = 0.0;
          L.fw_toff.push_back(int(fwt.size()));
          L.fw_goff.push_back(int(fwm.size()));
          for (int id : wv.blocked) {
            const Node& nd = P.nodes[id];
            if (!D->h_nodes[id].defer) continue;
            const int nblk = (nd.ni + 127) / 128;
            if (t >= nblk) continue;
            const int64_t M = nd.m_off, ldm = nd.ldm;
            const int k0 = t * 128, k1 = std::min(nd.ni, k0 + 128), bk = k1 - k0;
            for (auto [c0, c1] : segs(nd)) {
              const int ncy = c1 - c0;
              const int64_t Yc = M + (int64_t(nd.ni) + c0) * ldm;
              // left-looking: Y_k -= L[k0:k1, 0:k0] Y[0:k0] (one GEMM, K = k0: the same
              // subtractions in the same order as the right-looking block updates), then
              // Y_k <- L_kk^{-1} Y_k (unit lower)
              fwt.push_back(TrsmDesc{reinterpret_cast<const double*>(M + k0 + int64_t(k0) * ldm),
                                     reinterpret_cast<double*>(Yc + k0), int(ldm), int(ldm), bk, ncy});
              fwm.push_back(GemmDesc{reinterpret_cast<const double*>(M + k0), reinterpret_cast<const double*>(Yc),
                                     reinterpret_cast<double*>(Yc + k0), bk, ncy, k0, int(ldm), int(ldm), int(ldm)});
              tiles = std::max(tiles, gemm_tiles(bk, ncy));
              mc = std::max(mc, ncy);
              fl += double(bk) * bk * ncy + 2.0 * double(bk) * ncy * k0;
              ++cnt;
            }
            kk = std::max(kk, k0);
          }
          L.fw_n.push_back(cnt);
          L.fw_tiles.push_back(tiles);
          L.fw_k.push_back(kk);
          L.fw_cols.push_back(mc);
          L.fw_flops.push_back(fl);
        }
      }
      L.copy_base = int(cd.size());
      for (int t = 0; t < maxblk; ++t) {
        const int off = int(gd.size()), toff = int(trs.size()), soff = int(gs.size());
        int cnt = 0, t1 = 0, t2 = 0, kk = 0, mc = 0;
        double fl = 0.0;
        std::vector<GemmDesc> g2;
        for (int id : wv.blocked) {
          const Node& nd = P.nodes[id];
          const int nblk = (nd.ni + 127) / 128;
          const int sblk = nblk - 1 - t;
          if (sblk < 0) continue;
          const int64_t M = nd.m_off, ldm = nd.ldm;
          const int k0 = sblk * 128, k1 = std::min(nd.ni, k0 + 128), bk = k1 - k0;
          for (auto [c0, c1] : segs(nd)) {
            const int ncy = c1 - c0;  // boundary columns + body-load columns (this segment)
            const int64_t Yc = M + (int64_t(nd.ni) + c0) * ldm;
            // substitution variant: Y_k <- U_kk^{-1} Y_k in place, Y[0:k0] -= U[0:k0, k0:k1] Y_k
            trs.push_back(TrsmDesc{reinterpret_cast<const double*>(M + k0 + int64_t(k0) * ldm),
                                   reinterpret_cast<double*>(Yc + k0), int(ldm), int(ldm), bk, ncy});
            gs.push_back(GemmDesc{reinterpret_cast<const double*>(M + int64_t(k0) * ldm),
                                  reinterpret_cast<const double*>(Yc + k0), reinterpret_cast<double*>(Yc), k0, ncy, bk,
                                  int(ldm), int(ldm), int(ldm)});
            // default (explicit block inverse): T = Uinv_k Y_k; Y[0:k0] -= U[0:k0, k0:k1] T; Y_k = T
            const int64_t uinv = nd.uinv_off + int64_t(sblk) * 2 * 128 * 128 + 128 * 128;
            gd.push_back(GemmDesc{reinterpret_cast<const double*>(uinv), reinterpret_cast<const double*>(Yc + k0),
                                  reinterpret_cast<double*>(nd.t_off), bk, ncy, bk, 128, int(ldm), 128});
            g2.push_back(GemmDesc{reinterpret_cast<const double*>(M + int64_t(k0) * ldm),
                                  reinterpret_cast<const double*>(nd.t_off), reinterpret_cast<double*>(Yc), k0, ncy, bk,
                                  int(ldm), 128, int(ldm)});
            cd.push_back(CopyDesc{reinterpret_cast<const double*>(nd.t_off), reinterpret_cast<double*>(Yc + k0), 128,
                                  int(ldm), bk, ncy});
            t1 = std::max(t1, gemm_tiles(bk, ncy));
            t2 = std::max(t2, gemm_tiles(std::max(k0, 1), ncy));
            mc = std::max(mc, ncy);
            fl += double(bk) * bk * ncy + 2.0 * k0 * double(ncy) * bk;
            ++cnt;
          }
          kk = std::max(kk, bk);
        }
        gd.insert(gd.end(), g2.begin(), g2.end());
        L.bs_off.push_back(off);
        L.bs_soff.push_back(soff);
        L.bs_tiles1.push_back(t1);
        L.bs_toff.push_back(toff);
        L.bs_cnt.push_back(cnt);
        L.bs_tiles2.push_back(t2);
        L.bs_k.push_back(kk);
        L.bs_cols.push_back(mc);
        L.bs_flops.push_back(fl);
      }
      L.fin_off = int(gd.size());
      L.fin_cnt = 0;
      for (int id : wv.blocked) {
        const Node& nd = P.nodes[id];
        const int64_t M = nd.m_off, ldm = nd.ldm;
        for (auto [c0, c1] : segs(nd)) {  // S and the body-load columns (dense_nd.cpp:181-184)
          const int ncy = c1 - c0;
          const int64_t Yc = M + (int64_t(nd.ni) + c0) * ldm;
          gd.push_back(GemmDesc{reinterpret_cast<const double*>(M + nd.ni), reinterpret_cast<const double*>(Yc),
                                reinterpret_cast<double*>(Yc + nd.ni), nd.sys_nb, ncy, nd.ni, int(ldm), int(ldm),
                                int(ldm)});
          L.fin_tiles = std::max(L.fin_tiles, gemm_tiles(nd.sys_nb, ncy));
          L.fin_flops += 2.0 * nd.sys_nb * double(ncy) * nd.ni;
          ++L.fin_cnt;
        }
        L.fin_k = std::max(L.fin_k, nd.ni);
        L.fin_aligned = L.fin_aligned && (nd.ni % 2 == 0);
        if (nd.colshard) L.gather_nodes.push_back(id);
      }
    }
    D->h_trs = std::move(trs);
    D->h_fw_copy = std::move(fwc);
    D->h_fw_gather = std::move(fwg);
    D->h_fw_trs = std::move(fwt);
    D->h_fw_gemm = std::move(fwm);
    D->gtmp_doubles = gtmp_need;
    D->subst_base = int(gd.size());
    gd.insert(gd.end(), gs.begin(), gs.end());
    D->h_bs_gemm = std::move(gd);
    D->h_bs_copy = std::move(cd);
    D->h_tri = std::move(td);
  }
  // compressed engine descriptors (arena offsets, relocated below)
  {
    auto off = [](int64_t o) { return reinterpret_cast<double*>(o); };
    auto coff = [](int64_t o) { return reinterpret_cast<const double*>(o); };
    for (size_t w = 0; w < P.waves.size(); ++w) {
      WaveLaunch& L = D->wl[w];
      const Wave& wv = P.waves[w];
      // structured merges: C (the reduced system's Schur complement) -> aligned copy,
      // T = -L_k C, S -= T R_k
      L.sm_copy = int(D->h_sm_copy.size());
      for (int id : wv.smerge) {
        const Node& nd = P.nodes[id];
        D->h_sm_copy.push_back(CopyDesc{coff(nd.m_off + nd.ni + int64_t(nd.ni) * nd.ldm), off(nd.cbuf_off), nd.ldm,
                                        nd.ldr, nd.sys_nb, nd.sys_nb});
      }
      L.sm_t = int(D->h_sg.size());
      for (int id : wv.smerge) {
        const Node& nd = P.nodes[id];
        D->h_sg.push_back(GemmDesc{coff(nd.lkg_off), coff(nd.cbuf_off), off(nd.tg_off), nd.nb, nd.sys_nb, nd.sys_nb,
                                   nd.ldg, nd.ldr, nd.ldg});
        L.sm_t_tiles = std::max(L.sm_t_tiles, gemm_tiles(nd.nb, nd.sys_nb));
        L.sm_t_k = std::max(L.sm_t_k, nd.sys_nb);
        L.sm_flops += 2.0 * nd.nb * double(nd.sys_nb) * nd.sys_nb;
      }
      L.sm_u = int(D->h_sg.size());
      for (int id : wv.smerge) {
        const Node& nd = P.nodes[id];
        D->h_sg.push_back(GemmDesc{coff(nd.tg_off), coff(nd.rkg_off), off(nd.s_off), nd.nb, nd.nb, nd.sys_nb, nd.ldg,
                                   nd.ldr, nd.ld});
        L.sm_u_tiles = std::max(L.sm_u_tiles, gemm_tiles(nd.nb, nd.nb));
        L.sm_u_k = std::max(L.sm_u_k, nd.sys_nb);
        L.sm_flops += 2.0 * nd.nb * double(nd.nb) * nd.sys_nb;
      }
      // factors of the wave's structured boxes (randomized range finder + Householder QR)
      // K-slice k of the sketches: rows [k0, k1) of Omega (k0 a multiple of 16); slice 0
      // into Y, slice s > 0 into the node's partials (summed afterwards, in slice order)
      auto kslice = [](const Node& nd, int sl, int* k0, int* k1) {
        const int kc = int(align_up((nd.nb + nd.ysplit - 1) / nd.ysplit, 16));
        *k0 = std::min(nd.nb, sl * kc);
        *k1 = std::min(nd.nb, *k0 + kc);
      };
      auto ypart = [](const Node& nd, int sl, int which) {  // which 0: Y1, 1: Y2
        if (sl == 0) return which ? nd.y2_off : nd.y1_off;
        return nd.ysp_off + (int64_t(sl - 1) * 2 + which) * nd.ldq * (nd.ell + kProbes);
      };
      L.cp_y1 = int(D->h_sg.size());
      for (int id : wv.compress) {
        const Node& nd = P.nodes[id];
        for (int sl = 0; sl < nd.ysplit; ++sl) {
          int k0, k1;
          kslice(nd, sl, &k0, &k1);
          D->h_sg.push_back(GemmDesc{coff(nd.s_off + nd.j0 + int64_t(k0) * nd.ld), coff(nd.om_off + k0),
                                     off(ypart(nd, sl, 0)), nd.jn, nd.ell + kProbes, k1 - k0, nd.ld, nd.ldf, nd.ldq});
          L.cp_y1_k = std::max(L.cp_y1_k, k1 - k0);
        }
        L.cp_y1_tiles = std::max(L.cp_y1_tiles, gemm_tiles(nd.jn, nd.ell + kProbes));
        L.cp_flops += 2.0 * nd.jn * double(nd.nb) * nd.ell;
      }
      L.cp_y1_n = int(D->h_sg.size()) - L.cp_y1;
      L.cp_lk = int(D->h_sg.size());
      for (int id : wv.compress) {
        const Node& nd = P.nodes[id];
        D->h_sg.push_back(GemmDesc{coff(nd.s_off + int64_t(nd.j0) * nd.ld), coff(nd.q2_off), off(nd.lk_off), nd.nb,
                                   nd.ell, nd.jn, nd.ld, nd.ldq, nd.ldf});
        L.cp_lk_tiles = std::max(L.cp_lk_tiles, gemm_tiles(nd.nb, nd.ell));
        L.cp_lk_k = std::max(L.cp_lk_k, nd.jn);
        L.cp_lk_aligned = L.cp_lk_aligned && ((nd.s_off + int64_t(nd.j0) * nd.ld) % 2 == 0) && (nd.ld % 2 == 0);
        L.cp_flops += 2.0 * nd.jn * double(nd.nb) * nd.ell;
      }
      L.cp_y2 = int(D->h_sg2.size());
      for (int id : wv.compress) {  // S[:, J]^T: row-major view of the J columns
        const Node& nd = P.nodes[id];
        for (int sl = 0; sl < nd.ysplit; ++sl) {
          int k0, k1;
          kslice(nd, sl, &k0, &k1);
          D->h_sg2.push_back(GemmDesc2{coff(nd.s_off + int64_t(nd.j0) * nd.ld + k0), nullptr, coff(nd.om_off + k0),
                                       off(ypart(nd, sl, 1)), nd.jn, nd.ell + kProbes, k1 - k0, nd.ld, 0,
                                       int(align_up(k1 - k0, 16)), k1 - k0, nd.ldf, nd.ldq});
        }
        L.cp_y2_tiles = std::max(L.cp_y2_tiles, gemm_tiles(nd.jn, nd.ell + kProbes));
        L.cp_flops += 2.0 * nd.jn * double(nd.nb) * nd.ell;
      }
      L.cp_y2_n = int(D->h_sg2.size()) - L.cp_y2;
      L.cp_sum = int(D->h_sum.size());
      for (int id : wv.compress) {
        const Node& nd = P.nodes[id];
        if (nd.ysplit < 2) continue;
        for (int which = 0; which < 2; ++which)
          D->h_sum.push_back(SumDesc{off(which ? nd.y2_off : nd.y1_off), coff(ypart(nd, 1, which)),
                                     2LL * nd.ldq * (nd.ell + kProbes), nd.ldq, nd.ldq, nd.jn, nd.ell + kProbes,
                                     nd.ysplit - 1});
        L.cp_sum_elems = std::max<long long>(L.cp_sum_elems, (long long)nd.jn * (nd.ell + kProbes));
      }
      L.cp_sum_n = int(D->h_sum.size()) - L.cp_sum;
      L.cp_rt = int(D->h_sg2.size());
      for (int id : wv.compress) {  // S[J, :]^T: row-major view of the J rows
        const Node& nd = P.nodes[id];
        D->h_sg2.push_back(GemmDesc2{coff(nd.s_off + nd.j0), nullptr, coff(nd.q1_off), off(nd.rt_off), nd.nb, nd.ell,
                                     nd.jn, nd.ld, 0, int(align_up(nd.jn, 16)), nd.jn, nd.ldq, nd.ldf});
        L.cp_rt_tiles = std::max(L.cp_rt_tiles, gemm_tiles(nd.nb, nd.ell));
        L.cp_flops += 2.0 * nd.jn * double(nd.nb) * nd.ell;
      }
      L.cp_qr = int(D->h_qr.size());
      for (int q = 0; q < 2; ++q)
        for (int id : wv.compress) {
          const Node& nd = P.nodes[id];
          D->h_qr.push_back(QrDesc{off(q ? nd.y2_off : nd.y1_off), off(q ? nd.q2_off : nd.q1_off),
                                   reinterpret_cast<double*>(int64_t(2 * D->h_qr.size())), coff(nd.s_off), nd.ldq,
                                   nd.ldq, nd.jn, nd.ell, kProbes, nd.ld, nd.nb, nd.nb - nd.jn});
          D->qr_node.push_back(id);
          L.cp_qr_m = std::max(L.cp_qr_m, nd.jn);
          L.cp_qr_n = std::max(L.cp_qr_n, nd.ell + kProbes);
          L.cp_flops += 8.0 * nd.jn * double(nd.ell) * nd.ell;  // factor + form Q
        }
    }
  }
  D->root_list_off = int(lists.size());
  lists.push_back(D->root_lu_node);
  D->h_lists = lists;
  // device buffers
  D->d_nodes = dalloc<NodeDev>(D->h_nodes.size());
  CK(cudaMemcpy(D->d_nodes, D->h_nodes.data(), D->h_nodes.size() * sizeof(NodeDev), cudaMemcpyHostToDevice));
  static_assert(sizeof(PosDev) == sizeof(PosEntry), "PosDev/PosEntry layout");
  D->d_pos = dalloc<PosDev>(P.pos.size());
  CK(cudaMemcpy(D->d_pos, P.pos.data(), P.pos.size() * sizeof(PosDev), cudaMemcpyHostToDevice));
  D->d_lists = dalloc<int>(lists.size());
  CK(cudaMemcpy(D->d_lists, lists.data(), lists.size() * sizeof(int), cudaMemcpyHostToDevice));
  D->d_arena = dalloc<double>(size_t(D->gtmp_doubles > 0 ? D->gtmp_off + D->gtmp_doubles
                                                           : D->lu_off + int64_t(D->ldlu) * nb));
  D->d_piv = dalloc<int>(size_t(P.piv_ints + align_up(nb, 4) + 260));
  if (P.key.nloads > 0) {
    D->d_load_col = dalloc<int>(size_t(D->nu));
    D->ldf = int(align_up(nb, 8));
    D->d_F = dalloc<double>(size_t(D->ldf) * P.key.nloads * 2);  // F, then the aligned copy of rhs_root
    const Node& rt = P.nodes[P.root];
    D->h_F_desc = GemmDesc{nullptr, D->d_F + size_t(D->ldf) * P.key.nloads, D->d_F, nb, P.key.nloads, nb, 0, D->ldf,
                           D->ldf};
    D->rhs_root_off = rt.rhs_off;
    D->rhs_root_ld = rt.rhs_ld;
    D->d_F_desc = dalloc<GemmDesc>(1);
  }
  {  // relocate the Schur-form descriptors (stored as arena offsets) and upload
    double* base = D->d_arena;
    auto rel = [&](auto* p) { return reinterpret_cast<decltype(p)>(base + reinterpret_cast<int64_t>(p)); };
    for (auto& g : D->h_bs_gemm) { g.A = rel(g.A); g.B = rel(g.B); g.C = rel(g.C); }
    for (auto& c : D->h_bs_copy) { c.src = rel(c.src); c.dst = rel(c.dst); }
    for (auto& t : D->h_tri) { t.LU = rel(t.LU); t.out = rel(t.out); }
    for (auto& t : D->h_trs) { t.U = rel(t.U); t.Y = rel(t.Y); }
    for (auto& c : D->h_fw_copy) { c.src = rel(c.src); c.dst = rel(c.dst); }
    for (auto& g : D->h_fw_gather) { g.src = rel(g.src); g.dst = rel(g.dst); }
    for (auto& t : D->h_fw_trs) { t.U = rel(t.U); t.Y = rel(t.Y); }
    for (auto& g : D->h_fw_gemm) { g.A = rel(g.A); g.B = rel(g.B); g.C = rel(g.C); }
    for (auto& c : D->h_sm_copy) { c.src = rel(c.src); c.dst = rel(c.dst); }
    for (auto& g : D->h_sg) { g.A = rel(g.A); g.B = rel(g.B); g.C = rel(g.C); }
    for (auto& g : D->h_sum) { g.dst = rel(g.dst); g.src = rel(g.src); }
    for (auto& g : D->h_sg2) { g.A = rel(g.A); g.B = rel(g.B); g.C = rel(g.C); }
    if (!D->h_qr.empty()) {
      D->d_qstat = dalloc<double>(2 * D->h_qr.size());
      CK(cudaMallocHost(&D->h_qstat, 2 * D->h_qr.size() * sizeof(double)));
    }
    for (auto& q : D->h_qr) {
      q.Y = rel(q.Y);
      q.Q = rel(q.Q);
      q.S = rel(q.S);
      q.stat = D->d_qstat + reinterpret_cast<int64_t>(q.stat);
    }
    auto upload_vec = [&](auto& h, auto*& d) {
      if (h.empty()) return;
      d = dalloc<std::remove_reference_t<decltype(h[0])>>(h.size());
      CK(cudaMemcpy(d, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    };
    upload_vec(D->h_fw_copy, D->d_fw_copy);
    upload_vec(D->h_fw_gather, D->d_fw_gather);
    upload_vec(D->h_fw_trs, D->d_fw_trs);
    upload_vec(D->h_fw_gemm, D->d_fw_gemm);
    D->tm_fw.build(D->h_fw_gemm);
    upload_vec(D->h_sm_copy, D->d_sm_copy);
    upload_vec(D->h_sg, D->d_sg);
    D->tm_sg.build(D->h_sg);
    upload_vec(D->h_sg2, D->d_sg2);
    upload_vec(D->h_sum, D->d_sum);
    upload_vec(D->h_qr, D->d_qr);
    D->d_eps = dalloc<double>(1);
    D->d_trs = dalloc<TrsmDesc>(D->h_trs.size());
    if (!D->h_trs.empty())
      CK(cudaMemcpy(D->d_trs, D->h_trs.data(), D->h_trs.size() * sizeof(TrsmDesc), cudaMemcpyHostToDevice));
    D->d_bs_gemm = dalloc<GemmDesc>(D->h_bs_gemm.size());
    D->d_bs_copy = dalloc<CopyDesc>(D->h_bs_copy.size());
    D->d_tri = dalloc<TriDesc>(D->h_tri.size());
    if (!D->h_bs_gemm.empty())
      CK(cudaMemcpy(D->d_bs_gemm, D->h_bs_gemm.data(), D->h_bs_gemm.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice));
    D->tm_bs.build(D->h_bs_gemm);
    if (!D->h_bs_copy.empty())
      CK(cudaMemcpy(D->d_bs_copy, D->h_bs_copy.data(), D->h_bs_copy.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    if (!D->h_tri.empty())
      CK(cudaMemcpy(D->d_tri, D->h_tri.data(), D->h_tri.size() * sizeof(TriDesc), cudaMemcpyHostToDevice));
  }
  D->d_pivstat = dalloc<double>(2 * D->h_nodes.size());
  {
    std::vector<int> chk(D->h_nodes.size(), 0);
    for (const Wave& wv : P.waves)
      for (const auto* lst : {&wv.micro, &wv.small, &wv.blocked})
        for (int id : *lst)
          if (P.nodes[id].ni > 0) chk[size_t(id)] = 1;
    if (size_t(D->root_lu_node) < chk.size()) chk[size_t(D->root_lu_node)] = 2;
    D->d_chk = dalloc<int>(chk.size());
    CK(cudaMemcpy(D->d_chk, chk.data(), chk.size() * sizeof(int), cudaMemcpyHostToDevice));
    D->d_bad = dalloc<int>(1);
    CK(cudaMallocHost(&D->h_bad, sizeof(int)));
  }
  D->d_stencil = dalloc<double>(size_t(5 * D->nu));
  D->lds = int(align_up(nb, 8));
  D->d_S = dalloc<double>(size_t(D->lds) * nb);
  D->ldg = int(align_up(nb, 8));
  if (P.key.world > 1) D->root_cw = (nb + P.key.world - 1) / P.key.world;
  // (collective: room for every rank's column chunk, gathered in place)
  D->d_G = dalloc<double>(size_t(D->ldg) * std::max<int64_t>(nb, int64_t(P.key.world) * D->root_cw));
  if (P.key.nloads > 0) {
    D->h_F_desc.A = D->d_G;
    D->h_F_desc.lda = D->ldg;
    CK(cudaMemcpy(D->d_F_desc, &D->h_F_desc, sizeof(GemmDesc), cudaMemcpyHostToDevice));
  }
  D->d_perm = dalloc<int>(nb);
  D->d_norm = dalloc<unsigned long long>(2);
  CK(cudaMallocHost(&D->h_pivstat, 2 * D->h_nodes.size() * sizeof(double)));
  CK(cudaMallocHost(&D->h_norm, 2 * sizeof(unsigned long long)));
  // Root inverse G = U^{-1} L^{-1} P (getri-style, 2 nb^3 flops) over 128-row
  // blocks with the diagonal-block solves deferred, so each sweep is a chain of
  // large GEMMs only: with L'_ik = L_ik Linv_kk and U'_ik = U_ik Uinv_kk
  // (one batched launch), the forward sweep on W = I is
  //   W[k1:, :k1] -= L'[k1:, k] W[k, :k1]      (W_k stays unsolved),
  // then Z_k = Linv_kk W_k for all k (batched), the backward sweep
  //   Z[:k0, :] -= U'[:k0, k] Z[k, :],
  // then W_k = Uinv_kk Z_k for all k (batched) and G = W P.
  // Descriptor ranges in h_inv_descs: [0, inv_pre) pre-products, then nblk - 1
  // forward, nblk Z solves, nblk - 1 backward, nblk final solves.
  const double* LU = D->d_arena + D->lu_off;
  D->d_W = dalloc<double>(size_t(D->ldg) * nb);
  D->d_LUp = dalloc<double>(size_t(D->ldlu) * nb);
  const int nblk = (nb + 127) / 128;
  D->d_tinv = dalloc<double>(size_t(nblk) * 2 * 128 * 128);
  auto tinv = [&](int kb_, int u) { return D->d_tinv + size_t(kb_) * 2 * 128 * 128 + (u ? 128 * 128 : 0); };
  for (int kb_ = 0; kb_ < nblk; ++kb_) {
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    if (nb - k1 > 0)
      D->h_inv_descs.push_back(GemmDesc{LU + k1 + int64_t(k0) * D->ldlu, tinv(kb_, 0),
                                        D->d_LUp + k1 + int64_t(k0) * D->ldlu, nb - k1, bk, bk, D->ldlu, 128, D->ldlu});
    if (k0 > 0)
      D->h_inv_descs.push_back(GemmDesc{LU + int64_t(k0) * D->ldlu, tinv(kb_, 1), D->d_LUp + int64_t(k0) * D->ldlu,
                                        k0, bk, bk, D->ldlu, 128, D->ldlu});
  }
  D->inv_pre = int(D->h_inv_descs.size());
  // diagonal-block inverses by substitution on identity blocks: Linv (unit
  // lower, forward) for every block, then Uinv (backward)
  for (int u = 0; u < 2; ++u)
    for (int kb_ = 0; kb_ < nblk; ++kb_) {
      const int k0 = kb_ * 128, bk = std::min(nb, k0 + 128) - k0;
      D->h_root_trs.push_back(TrsmDesc{LU + k0 + int64_t(k0) * D->ldlu, tinv(kb_, u), D->ldlu, 128, bk, bk});
    }
  D->d_root_trs = dalloc<TrsmDesc>(D->h_root_trs.size());
  CK(cudaMemcpy(D->d_root_trs, D->h_root_trs.data(), D->h_root_trs.size() * sizeof(TrsmDesc), cudaMemcpyHostToDevice));
  for (int kb_ = 0; kb_ + 1 < nblk; ++kb_) {  // forward
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{D->d_LUp + k1 + int64_t(k0) * D->ldlu, D->d_W + k0, D->d_W + k1, nb - k1, k1,
                                      bk, D->ldlu, D->ldg, D->ldg});
  }
  for (int kb_ = 0; kb_ < nblk; ++kb_) {  // Z_k = Linv_kk W_k (Z in the G buffer, zero beyond column k1)
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{tinv(kb_, 0), D->d_W + k0, D->d_G + k0, bk, k1, bk, 128, D->ldg, D->ldg});
  }
  for (int kb_ = 1; kb_ < nblk; ++kb_) {  // backward (used in reverse order)
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{D->d_LUp + int64_t(k0) * D->ldlu, D->d_G + k0, D->d_G, k0, nb, bk, D->ldlu,
                                      D->ldg, D->ldg});
  }
  for (int kb_ = 0; kb_ < nblk; ++kb_) {  // W_k = Uinv_kk Z_k
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{tinv(kb_, 1), D->d_G + k0, D->d_W + k0, bk, nb, bk, 128, D->ldg, D->ldg});
  }
  // Variant used by the build: U^{-1} formed on the side stream while the forward
  // sweep runs (the same deferred-solve backward sweep on I, upper-triangular column
  // ranges only), then W = U^{-1} Z as ONE batched GEMM over the 128-row blocks of
  // U^{-1} (block row I needs only K >= I) instead of nblk - 1 dependent updates.
  D->d_UI = dalloc<double>(size_t(D->ldg) * nb);
  D->d_UI2 = dalloc<double>(size_t(D->ldg) * nb);
  D->inv_ui = int(D->h_inv_descs.size());
  for (int kb_ = 1; kb_ < nblk; ++kb_) {  // UI[:k0, k0:] -= U'[:k0, k] UI[k, k0:] (used in reverse order)
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{D->d_LUp + int64_t(k0) * D->ldlu, D->d_UI + k0 + int64_t(k0) * D->ldg,
                                      D->d_UI + int64_t(k0) * D->ldg, k0, nb - k0, bk, D->ldlu, D->ldg, D->ldg});
  }
  for (int kb_ = 0; kb_ < nblk; ++kb_) {  // UI2_k = Uinv_kk UI_k (columns >= k0)
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{tinv(kb_, 1), D->d_UI + k0 + int64_t(k0) * D->ldg,
                                      D->d_UI2 + k0 + int64_t(k0) * D->ldg, bk, nb - k0, bk, 128, D->ldg, D->ldg});
  }
  for (int kb_ = 0; kb_ < nblk; ++kb_) {  // W[I] = UI2[I, I:] Z[I:, :]
    const int k0 = kb_ * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
    D->h_inv_descs.push_back(GemmDesc{D->d_UI2 + k0 + int64_t(k0) * D->ldg, D->d_G + k0, D->d_W + k0, bk, nb, nb - k0,
                                      D->ldg, D->ldg, D->ldg});
  }
  if (P.key.world > 1) {  // collective top build: G column chunks by block substitution
    const int cw = D->root_cw;
    for (int r = 0; r < P.key.world; ++r) {
      if (P.key.wrank >= 0 && r != P.key.wrank) continue;
      const int c0 = r * cw, c1 = std::min(nb, c0 + cw);
      if (c1 > c0) D->root_chunks.push_back({c0, c1});
    }
    double* G = D->d_G;
    const int ldg = D->ldg, ldl = D->ldlu;
    for (int t = 0; t < nblk; ++t) {  // forward, left-looking: G_k -= L[k, :k0] G[:k0]; G_k <- L_kk^{-1} G_k
      const int k0 = t * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
      D->rg_off.push_back(int(D->h_rg.size()));
      D->rt_off.push_back(int(D->h_rt.size()));
      for (auto [c0, c1] : D->root_chunks) {
        if (k0 > 0)
          D->h_rg.push_back(GemmDesc{LU + k0, G + int64_t(c0) * ldg, G + k0 + int64_t(c0) * ldg, bk, c1 - c0, k0, ldl,
                                     ldg, ldg});
        D->h_rt.push_back(TrsmDesc{LU + k0 + int64_t(k0) * ldl, G + k0 + int64_t(c0) * ldg, ldl, ldg, bk, c1 - c0});
      }
      D->rg_cnt.push_back(int(D->h_rg.size()) - D->rg_off.back());
      D->rt_cnt.push_back(int(D->h_rt.size()) - D->rt_off.back());
    }
    for (int t = nblk - 1; t >= 0; --t) {  // backward: G_k <- U_kk^{-1} G_k; G[:k0] -= U[:k0, k] G_k
      const int k0 = t * 128, k1 = std::min(nb, k0 + 128), bk = k1 - k0;
      D->rg_off.push_back(int(D->h_rg.size()));
      D->rt_off.push_back(int(D->h_rt.size()));
      for (auto [c0, c1] : D->root_chunks) {
        D->h_rt.push_back(TrsmDesc{LU + k0 + int64_t(k0) * ldl, G + k0 + int64_t(c0) * ldg, ldl, ldg, bk, c1 - c0});
        if (k0 > 0)
          D->h_rg.push_back(GemmDesc{LU + int64_t(k0) * ldl, G + k0 + int64_t(c0) * ldg, G + int64_t(c0) * ldg, k0,
                                     c1 - c0, bk, ldl, ldg, ldg});
      }
      D->rg_cnt.push_back(int(D->h_rg.size()) - D->rg_off.back());
      D->rt_cnt.push_back(int(D->h_rt.size()) - D->rt_off.back());
    }
    if (!D->h_rg.empty()) {
      D->d_rg = dalloc<GemmDesc>(D->h_rg.size());
      CK(cudaMemcpy(D->d_rg, D->h_rg.data(), D->h_rg.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice));
      D->tm_rg.build(D->h_rg);
    }
    D->d_rt = dalloc<TrsmDesc>(std::max<size_t>(D->h_rt.size(), 1));
    if (!D->h_rt.empty())
      CK(cudaMemcpy(D->d_rt, D->h_rt.data(), D->h_rt.size() * sizeof(TrsmDesc), cudaMemcpyHostToDevice));
  }
  D->d_inv_descs = dalloc<GemmDesc>(D->h_inv_descs.size());
  CK(cudaMemcpy(D->d_inv_descs, D->h_inv_descs.data(), D->h_inv_descs.size() * sizeof(GemmDesc),
                cudaMemcpyHostToDevice));
  D->tm_inv.build(D->h_inv_descs);
  D->ev_wave.resize(P.waves.size());
  for (auto& e : D->ev_wave) CK(cudaEventCreate(&e));
  CK(cudaEventCreate(&D->ev_start));
  CK(cudaEventCreate(&D->ev_root));
  CK(cudaEventCreate(&D->ev_end));
  CK(cudaEventCreateWithFlags(&D->ev_rp, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_rest, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_rest2[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_rest2[1], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_S, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_inv_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_inv_join, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&D->copy, cudaStreamNonBlocking));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&D->side, cudaStreamNonBlocking, lo));
  return D;
}

// Waves whose rank-32 updates of the boundary columns add up to at least this
// much work (sum of ni (ncols - ni)) defer those columns (NodeDev::defer): the
// right-looking updates stream the whole ni x total block from HBM every step;
// one blocked forward substitution after the LU (rank-128 GEMM updates, the
// same arithmetic in the same order: bitwise-identical S) cuts that traffic 4x.
// Lighter waves keep the look-ahead schedule (their boundary updates hide
// behind the latency-bound panel chain; deferring measured slower there).
// DTN_DEFER_MIN_WORK (0: never).
double defer_min_work() {
  static const double v = [] {
    const char* e = std::getenv("DTN_DEFER_MIN_WORK");
    const double x = e ? std::atof(e) : 3.2e7;
    return x <= 0.0 ? 1e300 : x;
  }();
  return v;
}

bool use_subst() {  // default: substitution (DTN_BACKSUB_SUBST=0 selects the explicit block inverses)
  const char* e = std::getenv("DTN_BACKSUB_SUBST");
  return !(e && e[0] == '0');
}

bool env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '1';
}

bool use_lookahead() {
  const char* e = std::getenv("DTN_NO_LOOKAHEAD");
  return !(e && e[0] == '1');
}

// One-CTA fused merges (k_fused.cu) for waves whose largest system has at least this many
// unknowns and fits one CTA's shared memory (DTN_FUSED_MERGE_MIN; 0 disables)
int fused_merge_min() {
  const char* e = std::getenv("DTN_FUSED_MERGE_MIN");
  return e ? std::atoi(e) : 64;
}

bool use_fused() {  // DTN_NO_FUSED=1: the unfused look-ahead (next-panel update on the main stream)
  const char* e = std::getenv("DTN_NO_FUSED");
  return use_lookahead() && !(e && e[0] == '1');
}

// Per-launch profiler (opts.profile): CUDA events around every launch,
// aggregated per kernel class with the algorithmic work of each launch.
enum KClass {
  K_SMALL = 0, K_GATHER, K_PANEL, K_ROWPANEL, K_TRAILING, K_BACKSUB, K_SCHUR, K_COPY, K_INV_TRSM, K_INV_GEMM, K_MISC,
  K_SUBST, K_SGATHER, K_SGEMM, K_COMPRESS, K_FUSED, K_COUNT
};
const char* kclass_name(int k) {
  static const char* names[K_COUNT] = {"small_elim", "gather",   "panel",    "rowpanel", "trailing_gemm", "backsub_gemm",
                                       "schur_gemm", "copy",     "inv_trsm", "inv_gemm", "misc", "backsub_subst",
                                       "struct_gather", "struct_gemm", "sketch_qr", "fused_merge"};
  return names[k];
}
struct Prof {
  struct Rec {
    int kclass;
    cudaEvent_t a, b;
    double flops, bytes;
    int wave;
  };
  std::vector<Rec> recs;
  int wave = -1;  // current wave (root inverse: number of waves)
  ~Prof() {
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
};

// All device work of one build, in stream order (captured into a graph).
void enqueue_build(PlanDev& D, cudaStream_t st, bool want_G, Prof* prof = nullptr, bool events = true) {
  const Plan& P = D.P;
  const KernelArgs a = D.args();
  int launches = 0;
  auto run_on = [&](cudaStream_t s_, int kclass, double flops, double bytes, auto&& fn) {
    Prof::Rec r{kclass, nullptr, nullptr, flops, bytes, prof ? prof->wave : -1};
    if (prof) {
      CK(cudaEventCreate(&r.a));
      CK(cudaEventCreate(&r.b));
      CK(cudaEventRecord(r.a, s_));
    }
    CK(fn());
    ++launches;
    if (prof) {
      CK(cudaEventRecord(r.b, s_));
      prof->recs.push_back(r);
    }
  };
  auto run = [&](int kclass, double flops, double bytes, auto&& fn) { run_on(st, kclass, flops, bytes, fn); };
  cudaStream_t st2 = D.side;
  // Blocked partial LU of a batch of systems with one-step look-ahead: after
  // panel(k) + rowpanel(k), the update of the next panel's columns runs on the
  // main stream (so panel(k+1) starts at once) while the rest of the trailing
  // update runs concurrently on the side stream; rowpanel(k+1) joins it.
  // schur: eliminate the interface rows only (trailing updates restricted to
  // rows [k1, ni), no boundary-row multipliers): leaves L\U of M_ii and
  // Y = L^{-1} P M_ib; the Schur complement is formed afterwards as
  // S = M_bb - M_bi (U^{-1} Y), the reference's association (dense_nd.cpp:181),
  // which is markedly more accurate than (M_bi U^{-1}) Y for the near-resonant
  // interface blocks of the Helmholtz configurations.
  auto blocked_lu = [&](const int* lst, const int* hlst, int cnt, int max_ni, int max_total, int max_nb, int kb,
                        bool swap_left, bool schur) {
    const int rows_lim = schur ? max_ni : 0;
    const int nb_rows = schur ? 0 : max_nb;
    // Fused look-ahead (no boundary rows in the panel columns: Schur merges
    // and the root LU): panel(s) applies step s-1 to its own columns in its
    // prologue, so the main stream runs only the panel chain; rowpanel(s) and
    // the trailing update of the remaining columns run on the side stream.
    // panel(s) waits for the side stream's step s-2 (its columns' updates).
    if (nb_rows == 0 && use_fused() && !panel_is_tall(max_ni)) {
      int s = 0;
      for (int k0 = 0; k0 < max_ni; k0 += kb, ++s) {
        double fp = 0.0, fr = 0.0, ft = 0.0;
        for (int i = 0; i < cnt; ++i) {
          const Node* ndp = hlst ? &P.nodes[hlst[i]] : nullptr;
          const double ni = ndp ? ndp->ni : max_ni;
          const double tot = ndp ? (D.h_nodes[hlst[i]].defer ? ndp->ni : ndp->total) : max_total;
          if (k0 >= ni) continue;
          const double kbe = std::min<double>(kb, ni - k0), mn = tot - k0 - kbe, mr = ni - k0 - kbe;
          fp += (ni - k0) * kbe * kbe;
          if (k0 > 0) fp += 2.0 * (ni - k0) * kb * kbe + kb * kb * kbe;  // prologue
          const double nn = std::min<double>(mr, kb);
          fr += kbe * kbe * (mn - nn);
          ft += 2.0 * mr * (mn - nn) * kbe;
        }
        if (s >= 2) CK(cudaStreamWaitEvent(st, D.ev_rest2[s & 1], 0));
        run(K_PANEL, fp, 0.0, [&] { return launch_panel(a, lst, cnt, max_ni - k0, k0, kb, st, true); });
        CK(cudaEventRecord(D.ev_rp, st));
        CK(cudaStreamWaitEvent(st2, D.ev_rp, 0));
        run_on(st2, K_ROWPANEL, fr, 0.0,
               [&] { return launch_rowpanel(a, lst, cnt, max_total, 0, k0, kb, swap_left, st2, true); });
        run_on(st2, K_TRAILING, ft, 0.0,
               [&] { return launch_trailing_update(a, lst, cnt, max_total, k0, kb, -1, 1 << 30, st2, max_ni); });
        CK(cudaEventRecord(D.ev_rest2[s & 1], st2));
      }
      if (s > 0) CK(cudaStreamWaitEvent(st, D.ev_rest2[(s - 1) & 1], 0));
      return;
    }
    bool pending = false;
    for (int k0 = 0; k0 < max_ni; k0 += kb) {
      double fp = 0.0, fr = 0.0, fn_ = 0.0, fr_ = 0.0;
      for (int i = 0; i < cnt; ++i) {
        const Node* ndp = hlst ? &P.nodes[hlst[i]] : nullptr;
        const double ni = ndp ? ndp->ni : max_ni, nbn = ndp ? ndp->nb : max_nb;
        const double tot = ndp ? (D.h_nodes[hlst[i]].defer ? ndp->ni : ndp->total) : max_total;
        if (k0 >= ni) continue;
        const double kbe = std::min<double>(kb, ni - k0), mn = tot - k0 - kbe;
        const double mr = schur ? ni - k0 - kbe : mn;  // rows of the trailing update
        fp += (ni - k0) * kbe * kbe;
        fr += kbe * kbe * ((schur ? 0.0 : nbn) + mn);
        const double nn = std::min<double>(mn, kb);
        fn_ += 2.0 * mr * nn * kbe;
        fr_ += 2.0 * mr * (mn - nn) * kbe;
      }
      const bool more = k0 + kb < max_ni;
      run(K_PANEL, fp, 0.0, [&] { return launch_panel(a, lst, cnt, max_ni - k0, k0, kb, st, false); });
      if (pending) CK(cudaStreamWaitEvent(st, D.ev_rest, 0));
      run(K_ROWPANEL, fr, 0.0,
          [&] { return launch_rowpanel(a, lst, cnt, max_total, nb_rows, k0, kb, swap_left, st, false); });
      if (more && use_lookahead()) {
        CK(cudaEventRecord(D.ev_rp, st));
        CK(cudaStreamWaitEvent(st2, D.ev_rp, 0));
        run(K_TRAILING, fn_, 0.0,
            [&] { return launch_trailing_update(a, lst, cnt, max_total, k0, kb, 0, kb, st, rows_lim); });
        run_on(st2, K_TRAILING, fr_, 0.0, [&] {
          return launch_trailing_update(a, lst, cnt, max_total, k0, kb, kb, 1 << 30, st2, rows_lim);
        });
        CK(cudaEventRecord(D.ev_rest, st2));
        pending = true;
      } else {
        run(K_TRAILING, fn_ + fr_, 0.0,
            [&] { return launch_trailing_update(a, lst, cnt, max_total, k0, kb, 0, 1 << 30, st, rows_lim); });
        pending = false;
      }
    }
    if (pending) CK(cudaStreamWaitEvent(st, D.ev_rest, 0));
  };
  auto list_flops = [&](const int* ids, int cnt) {
    double f = 0.0;
    for (int i = 0; i < cnt; ++i) f += merge_flop_count(P.nodes[ids[i]].ni, P.nodes[ids[i]].nb);
    return f;
  };
  const std::vector<int>& hl = D.h_lists;
  if (events) CK(cudaEventRecord(D.ev_start, st));
  for (size_t w = 0; w < D.wl.size(); ++w) {
    if (prof) prof->wave = int(w);
    const WaveLaunch& L = D.wl[w];
    if (L.micro_cnt)
      run(K_SMALL, list_flops(hl.data() + L.micro_off, L.micro_cnt), 0.0, [&] {
        return launch_small_elim(a, D.d_lists + L.micro_off, L.micro_cnt, L.micro_max, true, st);
      });
    // waves of many mid-size merges: the whole merge in one CTA's shared memory (k_fused.cu)
    auto fused_dims = [&](const int* ids, int cnt, int& mni, int& mnb, int& mtot) {
      mni = mnb = mtot = 0;
      bool ok = fused_merge_min() > 0 && P.key.nloads == 0;
      for (int i = 0; i < cnt && ok; ++i) {
        const Node& nd = P.nodes[ids[i]];
        ok = nd.kind == NodeKind::merge && !nd.smerge && nd.cw == 0 && nd.ni > 0 && nd.total > nd.ni;
        mni = std::max(mni, nd.ni);
        mnb = std::max(mnb, nd.total - nd.ni);
        mtot = std::max(mtot, nd.total);
      }
      return ok && mtot >= fused_merge_min() && fused_merge_fits(mni, mnb, mtot);
    };
    int f_ni = 0, f_nb = 0, f_tot = 0;
    if (L.small_cnt) {
      if (fused_dims(hl.data() + L.small_off, L.small_cnt, f_ni, f_nb, f_tot))
        run(K_FUSED, list_flops(hl.data() + L.small_off, L.small_cnt), 0.0, [&] {
          return launch_fused_merge(a, D.d_lists + L.small_off, L.small_cnt, f_ni, f_nb, f_tot, st);
        });
      else
        run(K_SMALL, list_flops(hl.data() + L.small_off, L.small_cnt), 0.0, [&] {
          return launch_small_elim(a, D.d_lists + L.small_off, L.small_cnt, L.small_max, false, st);
        });
    }
    if (L.blk_cnt && L.sm_cnt == 0 && L.gather_nodes.empty() && L.blk_cnt >= 16 &&
        fused_dims(hl.data() + L.blk_off, L.blk_cnt, f_ni, f_nb, f_tot)) {
      run(K_FUSED, list_flops(hl.data() + L.blk_off, L.blk_cnt), 0.0, [&] {
        return launch_fused_merge(a, D.d_lists + L.blk_off, L.blk_cnt, f_ni, f_nb, f_tot, st);
      });
    } else if (L.blk_cnt) {
      const int* lst = D.d_lists + L.blk_off;
      const int* hlst = hl.data() + L.blk_off;
      double gb = 0.0;
      for (int i = 0; i < L.blk_cnt; ++i) gb += 16.0 * double(P.nodes[hlst[i]].total) * P.nodes[hlst[i]].total;
      run(K_GATHER, 0.0, gb,
          [&] { return launch_gather(a, D.d_lists + L.gd_off, L.gd_cnt, L.gd_max_total, st); });
      if (L.sm_cnt)  // structured merges: the reduced interface system (Step 1)
        run(K_SGATHER, 0.0, 0.0,
            [&] { return launch_sgather_red(a, D.d_lists + L.sm_off, L.sm_cnt, L.sm_max_total, st); });
      // deferred boundary columns need L in the final row order (P A = L U): the row
      // moves of every step are then also applied to the factored columns (swap_left)
      blocked_lu(lst, hlst, L.blk_cnt, L.blk_max_ni, L.blk_max_total, L.blk_max_nb, L.kb, L.fw_cnt > 0, true);
      if (L.fw_cnt > 0) {  // deferred boundary columns: Y = L^{-1} P M_ib
        run(K_COPY, 0.0, 0.0, [&] { return launch_copy2d_batched(D.d_fw_copy + L.fw_copy_off, L.fw_cnt, st); });
        run(K_COPY, 0.0, 0.0,
            [&] { return launch_row_gather(D.d_fw_gather + L.fw_gather_off, L.fw_cnt, D.d_piv, st); });
        for (size_t t = 0; t < L.fw_n.size(); ++t) {
          if (t > 0)  // block 0 has no left part
            run(K_BACKSUB, L.fw_flops[t], 0.0, [&] {
              return gemm_go(D.d_fw_gemm, D.tm_fw, size_t(L.fw_goff[t]), L.fw_n[t], L.fw_tiles[t], L.fw_k[t], -1.0, 1.0, st, true);
            });
          run(K_SUBST, 0.0, 0.0, [&] {
            return launch_trsm_batched(D.d_fw_trs + L.fw_toff[t], L.fw_n[t], L.fw_cols[t], 128, true, st);
          });
        }
      }
      // X = U^{-1} Y by 128-row blocks from the bottom: dtrsm-style
      // substitution on the diagonal blocks (default; as accurate as the
      // reference on the near-resonant configurations) or explicit block
      // inverses (DTN_BACKSUB_SUBST=0; GEMM only), then S = M_bb - M_bi X
      if (!use_subst()) {
        run(K_INV_TRSM, 0.0, 0.0,
            [&] { return launch_tri_inv_u_batched(D.d_tri + L.tri_off, L.blk_cnt, L.tri_blocks, st); });
      }
      int coff = L.copy_base;
      for (size_t t = 0; t < L.bs_off.size(); ++t) {
        const int off = L.bs_off[t], cnt = L.bs_cnt[t];
        if (use_subst()) {
          run(K_SUBST, 0.0, 0.0,
              [&] {
                return env_flag("DTN_SUBST_REF")
                           ? launch_trsm_upper_ref(D.d_trs + L.bs_toff[t], cnt, L.bs_cols[t], st)
                           : launch_trsm_batched(D.d_trs + L.bs_toff[t], cnt, L.bs_cols[t], L.bs_k[t], false, st);
              });
          run(K_BACKSUB, L.bs_flops[t], 0.0, [&] {
            return gemm_go(D.d_bs_gemm, D.tm_bs, size_t(D.subst_base + L.bs_soff[t]), cnt, L.bs_tiles2[t], L.bs_k[t], -1.0, 1.0,
                           st, true);
          });
        } else {
          run(K_BACKSUB, 0.0, 0.0, [&] {
            return gemm_go(D.d_bs_gemm, D.tm_bs, size_t(off), cnt, L.bs_tiles1[t], L.bs_k[t], 1.0, 0.0, st, true);
          });
          run(K_BACKSUB, L.bs_flops[t], 0.0, [&] {
            return gemm_go(D.d_bs_gemm, D.tm_bs, size_t(off + cnt), cnt, L.bs_tiles2[t], L.bs_k[t], -1.0, 1.0, st, true);
          });
          run(K_COPY, 0.0, 0.0, [&] { return launch_copy2d_batched(D.d_bs_copy + coff, cnt, st); });
        }
        coff += cnt;
      }
      run(K_SCHUR, L.fin_flops, 0.0, [&] {
        return gemm_go(D.d_bs_gemm, D.tm_bs, size_t(L.fin_off), L.fin_cnt, L.fin_tiles, L.fin_k, -1.0, 1.0, st,
                       L.fin_aligned);
      });
      if (!L.gather_nodes.empty() && D.comm) {  // collective top build: every rank's column chunk to all
        const NcclApi& nc = nccl();
        nccl_check(nc.GroupStart(), "ncclGroupStart");
        for (int id : L.gather_nodes) {
          const Node& nd = P.nodes[id];
          double* Mb = D.d_arena + nd.m_off + int64_t(nd.ni) * nd.ldm;
          const size_t cnt = size_t(nd.ldm) * nd.cw;
          nccl_check(nc.AllGather(Mb + cnt * std::max(P.key.wrank, 0), Mb, cnt, ncclDouble,
                                  static_cast<ncclComm_t>(D.comm), st),
                     "ncclAllGather (merge columns)");
        }
        nccl_check(nc.GroupEnd(), "ncclGroupEnd");
      }
      if (L.sm_cnt) {  // Steps 2-3: S = M_kk + L_k C R_k
        const int* sl = D.d_lists + L.sm_off;
        run(K_SGATHER, 0.0, 0.0, [&] { return launch_kk_gather(a, sl, L.sm_cnt, L.sm_max_nb, st); });
        run(K_SGATHER, 0.0, 0.0, [&] { return launch_factor_gather(a, sl, L.sm_cnt, L.sm_max_elems, st); });
        run(K_COPY, 0.0, 0.0, [&] { return launch_copy2d_batched(D.d_sm_copy + L.sm_copy, L.sm_cnt, st); });
        run(K_SGEMM, L.sm_flops * 0.0, 0.0, [&] {
          return gemm_go(D.d_sg, D.tm_sg, size_t(L.sm_t), L.sm_cnt, L.sm_t_tiles, L.sm_t_k, -1.0, 0.0, st, true);
        });
        run(K_SGEMM, L.sm_flops, 0.0, [&] {
          return gemm_go(D.d_sg, D.tm_sg, size_t(L.sm_u), L.sm_cnt, L.sm_u_tiles, L.sm_u_k, -1.0, 1.0, st, true);
        });
      }
    }
    if (L.cp_cnt) {  // the wave's structured boxes: factors for their next merge
      const int* cl = D.d_lists + L.cp_off;
      run(K_COMPRESS, 0.0, 0.0, [&] { return launch_omega(a, cl, L.cp_cnt, L.cp_max_elems, st); });
      run(K_SGEMM, 0.0, 0.0, [&] {
        return launch_gemm_desc(D.d_sg + L.cp_y1, L.cp_y1_n, L.cp_y1_tiles, L.cp_y1_k, 1.0, 0.0, st, false);
      });
      run(K_SGEMM, 0.0, 0.0,
          [&] { return launch_gemm_desc2(D.d_sg2 + L.cp_y2, L.cp_y2_n, L.cp_y2_tiles, false, st); });
      if (L.cp_sum_n)
        run(K_SGATHER, 0.0, 0.0,
            [&] { return launch_sum_partials(D.d_sum + L.cp_sum, L.cp_sum_n, L.cp_sum_elems, st); });
      run(K_COMPRESS, 0.0, 0.0,
          [&] { return launch_hqr(D.d_qr + L.cp_qr, 2 * L.cp_cnt, L.cp_qr_m, L.cp_qr_n, D.d_eps, st); });
      run(K_SGEMM, 0.0, 0.0,
          [&] { return launch_gemm_desc2(D.d_sg2 + L.cp_rt, L.cp_cnt, L.cp_rt_tiles, false, st); });
      run(K_SGEMM, L.cp_flops, 0.0, [&] {
        return gemm_go(D.d_sg, D.tm_sg, size_t(L.cp_lk), L.cp_cnt, L.cp_lk_tiles, L.cp_lk_k, 1.0, 0.0, st, L.cp_lk_aligned);
      });
    }
    if (events) CK(cudaEventRecord(D.ev_wave[w], st));
  }
  // compact copy of the root S
  const Node& root = P.nodes[P.root];
  const double* Sview = D.d_arena + root.s_off;
  const double nb2 = double(D.nb) * D.nb;
  run(K_COPY, 0.0, 16.0 * nb2, [&] { return launch_copy2d(Sview, root.ld, D.d_S, D.lds, D.nb, D.nb, st); });
  // (external event: a host-side export of S can overlap the root inverse)
  {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    CK(cudaEventRecordWithFlags(D.ev_S, st,
                                cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault));
  }
  if (events) CK(cudaEventRecord(D.ev_root, st));
  if (prof) prof->wave = int(D.wl.size());
  if (want_G) {
    const int nb = D.nb;
    panel_kb(nb);  // throws beyond the tall panel's rows
    double* LU = D.d_arena + D.lu_off;
    run(K_COPY, 0.0, 16.0 * nb2, [&] { return launch_copy2d(D.d_S, D.lds, LU, D.ldlu, nb, nb, st); });
    const int* rl = D.d_lists + D.root_list_off;
    blocked_lu(rl, nullptr, 1, nb, nb, 0, D.root_kb, true, false);
    // the panels maintain perm[pos] = original row of the root LU (P A = L U)
    const int* perm = D.d_piv + D.h_nodes[D.root_lu_node].piv_off;
    if (P.key.world > 1) {  // collective top build: this rank's column chunk of G, gathered
      const int nblk = (nb + 127) / 128, mb = std::min(nb, 128);
      for (auto [c0, c1] : D.root_chunks)
        run(K_MISC, 0.0, 8.0 * nb * (c1 - c0), [&] {
          return launch_perm_identity_cols(perm, nb, c0, c1 - c0, D.d_G + int64_t(c0) * D.ldg, D.ldg, st);
        });
      int maxc = 0;
      for (auto [c0, c1] : D.root_chunks) maxc = std::max(maxc, c1 - c0);
      for (int q = 0; q < 2 * nblk; ++q) {
        const bool fwd = q < nblk;
        auto gem = [&] {
          if (D.rg_cnt[q] == 0) return;
          int tiles = 0, kmax = 0;
          double f = 0.0;
          for (int i = D.rg_off[q]; i < D.rg_off[q] + D.rg_cnt[q]; ++i) {
            const GemmDesc& g = D.h_rg[i];
            tiles = std::max(tiles, gemm_tiles(g.m, g.n));
            kmax = std::max(kmax, g.k);
            f += 2.0 * g.m * g.n * g.k;
          }
          run(K_INV_GEMM, f, 0.0, [&] {
            return gemm_go(D.d_rg, D.tm_rg, size_t(D.rg_off[q]), D.rg_cnt[q], tiles, kmax, -1.0, 1.0, st, true);
          });
        };
        auto trs = [&] {
          run(K_INV_TRSM, 0.0, 0.0, [&] {
            return launch_trsm_batched(D.d_rt + D.rt_off[q], D.rt_cnt[q], maxc, mb, fwd, st);
          });
        };
        if (fwd) {
          gem();
          trs();
        } else {
          trs();
          gem();
        }
      }
      if (D.comm) {
        const size_t cnt = size_t(D.ldg) * D.root_cw;
        nccl_check(nccl().AllGather(D.d_G + cnt * std::max(P.key.wrank, 0), D.d_G, cnt, ncclDouble,
                                    static_cast<ncclComm_t>(D.comm), st),
                   "ncclAllGather (G columns)");
      }
      CK(cudaMemsetAsync(D.d_norm, 0, 2 * sizeof(unsigned long long), st));
      run(K_MISC, 0.0, 8.0 * nb2, [&] { return launch_norm1(D.d_S, D.lds, nb, nb, D.d_norm, st); });
      run(K_MISC, 0.0, 8.0 * nb2, [&] { return launch_norm1(D.d_G, D.ldg, nb, nb, D.d_norm + 1, st); });
      if (events) CK(cudaEventRecord(D.ev_end, st));
      D.launches = launches;
      return;
    }
    if (env_flag("DTN_TRIINV_REF")) {
      run(K_INV_TRSM, 0.0, 0.0, [&] { return launch_tri_inv_blocks(LU, D.ldlu, nb, D.d_tinv, st); });
    } else {
      const int nblk = (nb + 127) / 128, mb = std::min(nb, 128);
      run(K_MISC, 0.0, 0.0, [&] { return launch_block_identity(D.d_tinv, 2 * nblk, st); });
      run(K_INV_TRSM, double(nb) * 128 * 128 / 3.0, 0.0,
          [&] { return launch_trsm_batched(D.d_root_trs, nblk, mb, mb, true, st); });
      run(K_INV_TRSM, double(nb) * 128 * 128 / 3.0, 0.0,
          [&] { return launch_trsm_batched(D.d_root_trs + nblk, nblk, mb, mb, false, st); });
    }
    run(K_MISC, 0.0, 8.0 * nb2, [&] { return launch_set_identity(D.d_W, D.ldg, nb, st); });
    const int nblk = (nb + 127) / 128;
    // a batch of descriptors [d0, d0 + cnt) in one launch
    auto gemm = [&](int d0, int cnt, double alpha, double beta) {
      if (cnt <= 0) return;
      int tiles = 0;
      double f = 0.0;
      for (int i = d0; i < d0 + cnt; ++i) {
        const GemmDesc& g = D.h_inv_descs[i];
        tiles = std::max(tiles, gemm_tiles(g.m, g.n));
        f += 2.0 * g.m * g.n * g.k;
      }
      run(K_INV_GEMM, f, 0.0, [&] {
        return gemm_go(D.d_inv_descs, D.tm_inv, size_t(d0), cnt, tiles, 128, alpha, beta, st, true);
      });
    };
    gemm(0, D.inv_pre, 1.0, 0.0);  // L' and U'
    int d = D.inv_pre;
    const bool ui_side = !env_flag("DTN_INV_SWEEP");
    if (ui_side) {  // U^{-1} on the side stream, concurrent with the forward sweep
      CK(cudaEventRecord(D.ev_inv_fork, st));
      CK(cudaStreamWaitEvent(st2, D.ev_inv_fork, 0));
      run_on(st2, K_MISC, 0.0, 8.0 * nb2, [&] { return launch_set_identity(D.d_UI, D.ldg, nb, st2); });
      CK(cudaMemsetAsync(D.d_UI2, 0, size_t(D.ldg) * nb * sizeof(double), st2));
      auto gemm2 = [&](int d0, int cnt, double alpha, double beta) {
        int tiles = 0;
        double f = 0.0;
        for (int i = d0; i < d0 + cnt; ++i) {
          const GemmDesc& g = D.h_inv_descs[i];
          tiles = std::max(tiles, gemm_tiles(g.m, g.n));
          f += 2.0 * g.m * g.n * g.k;
        }
        run_on(st2, K_INV_GEMM, f, 0.0,
               [&] { return gemm_go(D.d_inv_descs, D.tm_inv, size_t(d0), cnt, tiles, 128, alpha, beta, st2, true); });
      };
      for (int kb_ = nblk - 1; kb_ >= 1; --kb_) gemm2(D.inv_ui + kb_ - 1, 1, -1.0, 1.0);
      gemm2(D.inv_ui + nblk - 1, nblk, 1.0, 0.0);  // UI2_k = Uinv_kk UI_k
      CK(cudaEventRecord(D.ev_inv_join, st2));
    }
    for (int kb_ = 0; kb_ + 1 < nblk; ++kb_) gemm(d + kb_, 1, -1.0, 1.0);  // forward sweep
    d += nblk - 1;
    CK(cudaMemsetAsync(D.d_G, 0, size_t(D.ldg) * nb * sizeof(double), st));
    gemm(d, nblk, 1.0, 0.0);  // Z_k = Linv_kk W_k
    d += nblk;
    if (ui_side) {
      CK(cudaStreamWaitEvent(st, D.ev_inv_join, 0));
      // W = U^{-1} Z: one batched launch, block row I with K = nb - 128 I
      int tiles = 0;
      double f = 0.0;
      const int f0 = D.inv_ui + (nblk - 1) + nblk;
      for (int i = f0; i < f0 + nblk; ++i) {
        const GemmDesc& g = D.h_inv_descs[i];
        tiles = std::max(tiles, gemm_tiles(g.m, g.n));
        f += 2.0 * g.m * g.n * g.k;
      }
      run(K_INV_GEMM, f, 0.0,
          [&] { return gemm_go(D.d_inv_descs, D.tm_inv, size_t(f0), nblk, tiles, nb, 1.0, 0.0, st, true); });
    } else {
      for (int kb_ = nblk - 1; kb_ >= 1; --kb_) gemm(d + kb_ - 1, 1, -1.0, 1.0);  // backward sweep
      d += nblk - 1;
      gemm(d, nblk, 1.0, 0.0);  // W_k = Uinv_kk Z_k
    }
    run(K_COPY, 0.0, 16.0 * nb2, [&] { return launch_permute_columns(D.d_W, D.ldg, perm, nb, D.d_G, D.ldg, st); });
    CK(cudaMemsetAsync(D.d_norm, 0, 2 * sizeof(unsigned long long), st));
    run(K_MISC, 0.0, 8.0 * nb2, [&] { return launch_norm1(D.d_S, D.lds, nb, nb, D.d_norm, st); });
    run(K_MISC, 0.0, 8.0 * nb2, [&] { return launch_norm1(D.d_G, D.ldg, nb, nb, D.d_norm + 1, st); });
    if (P.key.nloads > 0) {  // body map F = G * rhs_root (accel_nd.cpp:872-875)
      const int nl = P.key.nloads;
      run(K_COPY, 0.0, 16.0 * nb * nl, [&] {
        return launch_copy2d(D.d_arena + D.rhs_root_off, D.rhs_root_ld, D.d_F + size_t(D.ldf) * nl, D.ldf, nb, nl, st);
      });
      run(K_INV_GEMM, 2.0 * nb2 * nl, 0.0,
          [&] { return launch_gemm_desc(D.d_F_desc, 1, gemm_tiles(nb, nl), nb, 1.0, 0.0, st, true); });
    }
  }
  if (events) CK(cudaEventRecord(D.ev_end, st));
  D.launches = launches;
}

bool use_graphs() {
  const char* e = std::getenv("DTN_NO_GRAPH");
  return !(e && e[0] == '1');
}

}  // namespace

struct dtn_ctx {
  // every call on a context (and on the operators built with it) runs under this
  // lock: the stream, cached plans, apply staging and the HBS apply workspaces
  // are shared state (recursive: the compressed build calls the other entries)
  std::recursive_mutex mu;
  int device = 0;
  // structured merges: factor ranks learned per problem family (dtn_gpu_build)
  std::map<std::string, std::vector<std::pair<int, int>>> learned_ranks;
  // multi-GPU (one process per GPU): this rank of `world`, the NCCL communicator
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  double* d_gather = nullptr;  // shard-S gather buffer (world x slot doubles)
  size_t gather_cap = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::vector<std::unique_ptr<PlanDev>> plans;
  std::string err;
  // apply staging
  double* d_x = nullptr;
  double* d_y = nullptr;
  size_t stage_cap = 0;
  double* d_skinny = nullptr;  // split-K partials of the small-batch apply
  size_t skinny_cap = 0;
  GemmDesc* d_desc = nullptr;
};

struct dtn_hbs {
  dtn_ctx* ctx = nullptr;
  std::unique_ptr<HbsDev> h;
};

struct dtn_op {
  std::vector<dtn_kernel_stats> kstats;
  dtn_ctx* ctx = nullptr;
  PlanDev* plan = nullptr;
  int nb = 0;
  bool has_G = false;
  double cond = 0.0;
  dtn_build_stats stats{};
  std::vector<dtn_level_stats> levels;
};

namespace {

thread_local std::string g_err;  // errors with no context (dtn_gpu_create)

template <class F>
int guarded(dtn_ctx* ctx, F&& f) {
  std::unique_lock<std::recursive_mutex> lock;
  if (ctx) lock = std::unique_lock<std::recursive_mutex>(ctx->mu);
  std::string& err = ctx ? ctx->err : g_err;
  (void)cudaGetLastError();  // drop stale non-sticky errors from unrelated runtime calls
  try {
    f();
    err.clear();
    return DTN_OK;
  } catch (const Singular& e) {
    err = e.what();
    return DTN_ESINGULAR;
  } catch (const HbsSingular& e) {
    err = e.what();
    return DTN_ESINGULAR;
  } catch (const std::invalid_argument& e) {
    err = e.what();
    return DTN_EINVAL;
  } catch (const std::domain_error& e) {
    err = e.what();
    return DTN_EINVAL;
  } catch (const std::exception& e) {
    err = e.what();
    return DTN_ECUDA;
  }
}

std::string label_of(const Plan& P, const Node& nd) {
  if (nd.label_level >= 0)
    return "interface block is singular [level " + std::to_string(nd.label_level) + " box " +
           std::to_string(nd.label_box) + "]";
  return "interior block A_ii is singular [leaf box " + std::to_string(nd.label_box) + "]";
}

bool pivots_ok(double pmin, double pmax) { return (pmin > pmax * 1e-300) && std::isfinite(pmax); }

}  // namespace

extern "C" {

int dtn_gpu_create(dtn_ctx** out, int device) {
  return guarded(nullptr, [&] {
    if (!out) throw std::invalid_argument("dtn_gpu_create: null output");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw CudaFail("dtn_gpu_create: no such CUDA device");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaFail("dtn_gpu_create: sm_100a (B200) device required");
    CK(cudaSetDevice(device));
    CK(gemm_init());
    CK(gemm_tma_init());
    CK(fused_init());
    CK(blocked_init());
    CK(misc_init());
    CK(hbs_kernels_init());
    CK(struct_init());
    auto* c = new dtn_ctx;
    c->device = device;
    CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    CK(cudaMalloc(&c->d_desc, 512));  // one descriptor + (at byte 256) its two tensor maps
    *out = c;
  });
}

int dtn_gpu_nccl_unique_id(uint8_t* id) {
  return guarded(nullptr, [&] {
    if (!id) throw std::invalid_argument("dtn_gpu_nccl_unique_id: null output");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, u.internal, 128);
  });
}

int dtn_gpu_create_rank(dtn_ctx** out, int device, int nranks, int rank, const uint8_t* id) {
  if (!out) return DTN_EINVAL;
  int rc = dtn_gpu_create(out, device);
  if (rc != DTN_OK || nranks < 1 || (nranks == 1 && !id)) return rc;
  dtn_ctx* c = *out;
  rc = guarded(c, [&] {
    if (rank < 0 || rank >= nranks || !id) throw std::invalid_argument("dtn_gpu_create_rank: bad rank or id");
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    CK(cudaSetDevice(device));
    nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->world = nranks;
    c->rank = rank;
  });
  if (rc != DTN_OK) {
    dtn_gpu_destroy(c);
    *out = nullptr;
  }
  return rc;
}

void dtn_gpu_destroy(dtn_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->plans.clear();
  if (ctx->comm) nccl().CommDestroy(ctx->comm);
  if (ctx->d_gather) cudaFree(ctx->d_gather);
  if (ctx->d_x) cudaFree(ctx->d_x);
  if (ctx->d_y) cudaFree(ctx->d_y);
  if (ctx->d_desc) cudaFree(ctx->d_desc);
  if (ctx->d_skinny) pool_free(ctx->d_skinny);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
}

const char* dtn_gpu_last_error(const dtn_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

unsigned long long dtn_gpu_hbs_launch_count(void) { return g_hbs_launches.load(); }

int dtn_gpu_set_stream(dtn_ctx* ctx, void* stream) {
  if (!ctx) return DTN_EINVAL;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return DTN_OK;
}

}  // extern "C"

namespace {

// world > 1: the top-of-tree build (opts->shard == -1, nshards == world) with its blocked
// merges column-sharded (PlanKey::world, wrank; comm != null: this rank's chunk plus
// ncclAllGather after each wave, comm == null: every chunk on this device)
int build_impl(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts,
               const std::vector<std::pair<int, int>>& ell_over, dtn_op** out, int world = 1, int wrank = -1,
               void* comm = nullptr) {
  return guarded(ctx, [&] {
    if (!ctx || !prob || !opts || !out) throw std::invalid_argument("dtn_gpu_build: null argument");
    if (prob->n < 4) throw std::invalid_argument("discretize: n must be >= 4");
    if (!prob->stencil) throw std::invalid_argument("dtn_gpu_build: null stencil");
    if (opts->engine != 0 && opts->engine != 1)
      throw std::invalid_argument("dtn_gpu_build: engine must be 0 (dense) or 1 (structured merges)");
    CK(cudaSetDevice(ctx->device));
    PlanKey key;
    key.n = prob->n;
    key.n_leaf = opts->n_leaf;
    key.leaf_side = opts->leaf_side;
    key.micro_max = opts->micro_max > 0 ? opts->micro_max : kDefaultMicro;
    key.small_max = kSmallMax;
    key.nshards = opts->nshards > 0 ? opts->nshards : 1;
    key.shard = opts->shard;
    if (key.nshards == 1) key.shard = -1;
    key.nloads = int(opts->nloads);
    key.keep = opts->keep_boxes ? 1 : 0;
    if (world > 1) {
      if (key.nshards != world || key.shard != -1) throw std::logic_error("collective top build: bad shard key");
      key.world = world;
      key.wrank = wrank;
    }
    if (opts->engine == 1) {  // compressed engine: structured merges above the crossover
      if (opts->nloads > 0)
        throw std::invalid_argument("dtn_gpu_build: body loads ride through the dense merges (engine 0)");
      if (opts->crossover < 1) throw std::invalid_argument("dtn_gpu_build: crossover must be >= 1");
      key.structured = 1;
      key.crossover = opts->crossover;
      key.ell_base = opts->rank_base > 0 ? opts->rank_base : 64;
      key.ell_step = opts->rank_step > 0 ? opts->rank_step : 8;
      key.ell_over = ell_over;
    }
    if (opts->nloads < 0 || (opts->nloads > 0 && !opts->load_ids))
      throw std::invalid_argument("dtn_gpu_build: bad body-load list");
    if (key.nloads > 0 && key.nshards > 1)
      throw std::invalid_argument("dtn_gpu_build: body loads are not supported in sharded builds");
    // (without G the body map is not formed; the root's reduced load columns are
    // read with dtn_gpu_root_rhs -- the compressed engine applies G_hbs to them)
    const bool top_mode = key.nshards > 1 && key.shard < 0;
    if (top_mode && !prob->shard_S) throw std::invalid_argument("dtn_gpu_build: top build needs the shard S blocks");
    if (key.leaf_side <= 0 && key.n_leaf < 16) throw std::invalid_argument("build_tree: n_leaf must be >= 16");
    PlanDev* D = nullptr;
    for (auto& p : ctx->plans)
      if (!p->busy && p->P.key == key) D = p.get();
    if (!D) {
      ctx->plans.push_back(make_plandev(key, ctx->device));
      D = ctx->plans.back().get();
    }
    D->comm = comm;
    cudaStream_t st = ctx->stream;
    const bool want_G = opts->want_G != 0 && key.shard < 0;  // a shard's S is not inverted
    if (top_mode) {
      const Plan& P0 = D->P;
      for (size_t i = 0; i < P0.inputs.size(); ++i) {
        const Node& nd = P0.nodes[P0.inputs[i]];
        if (!prob->shard_S[i]) throw std::invalid_argument("dtn_gpu_build: null shard S");
        CK(cudaMemcpy2DAsync(D->d_arena + nd.s_off, size_t(nd.ld) * 8, prob->shard_S[i], size_t(nd.nb) * 8,
                             size_t(nd.nb) * 8, size_t(nd.nb),
                             prob->shard_S_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
      }
    }
    const bool profile = opts->profile != 0;
    std::unique_ptr<Prof> prof;
    CK(cudaMemcpyAsync(D->d_stencil, prob->stencil, size_t(5 * D->nu) * sizeof(double),
                       prob->stencil_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    const double eps = opts->epsilon > 0.0 ? opts->epsilon : 1e-10;  // numerical-rank threshold of the factors
    CK(cudaMemcpyAsync(D->d_eps, &eps, sizeof(double), cudaMemcpyHostToDevice, st));
    if (key.nloads > 0) {  // LoadPanel (dense_nd.hpp:29-32): unit loads, distinct strictly-interior unknowns
      std::vector<int> col(size_t(D->nu), -1);
      const int s_ = key.n - 2;
      for (int j = 0; j < key.nloads; ++j) {
        const int64_t id = opts->load_ids[j];
        if (id < 0 || id >= D->nu) throw std::invalid_argument("load node is outside the grid");
        const int x = int(id % s_) + 1, y = int(id / s_) + 1;
        if (x == 1 || y == 1 || x == s_ || y == s_)
          throw std::invalid_argument("load node (" + std::to_string(x) + ", " + std::to_string(y) +
                                      ") is not strictly interior to the root box");
        if (col[size_t(id)] >= 0)
          throw std::invalid_argument("duplicate load node (" + std::to_string(x) + ", " + std::to_string(y) + ")");
        col[size_t(id)] = j;
      }
      CK(cudaMemcpy(D->d_load_col, col.data(), col.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    if (profile) {
      prof = std::make_unique<Prof>();
      enqueue_build(*D, st, want_G, prof.get());
    } else if (use_graphs() && !comm) {  // (collective builds enqueue NCCL calls directly)
      if (!D->gexec || D->graph_want_G != int(want_G)) {
        if (D->gexec) {
          CK(cudaGraphExecDestroy(D->gexec));
          D->gexec = nullptr;
        }
        cudaStream_t cap;
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&cap, cudaStreamNonBlocking, hi));
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue_build(*D, cap, want_G, nullptr, false);
        } catch (...) {
          cudaStreamEndCapture(cap, &g);
          cudaStreamDestroy(cap);
          throw;
        }
        CK(cudaStreamEndCapture(cap, &g));
        CK(cudaGraphInstantiateWithFlags(&D->gexec, g, cudaGraphInstantiateFlagUseNodePriority));
        CK(cudaGraphDestroy(g));
        CK(cudaStreamDestroy(cap));
        D->graph_want_G = int(want_G);
      }
      const auto hl0 = std::chrono::steady_clock::now();
      CK(cudaEventRecord(D->ev_start, st));
      CK(cudaGraphLaunch(D->gexec, st));
      CK(cudaEventRecord(D->ev_end, st));
      if (std::getenv("DTN_TRACE_BUILD"))
        std::fprintf(stderr, "[build] graph launch (host) %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hl0).count());
    } else {
      enqueue_build(*D, st, want_G);
    }
    if (opts->export_S) {  // S to the caller while the root inverse runs
      if (opts->export_lds < D->nb) throw std::invalid_argument("dtn_gpu_build: export_lds < nb");
      CK(cudaStreamWaitEvent(D->copy, D->ev_S, 0));
      CK(cudaMemcpy2DAsync(opts->export_S, size_t(opts->export_lds) * 8, D->d_S, size_t(D->lds) * 8,
                           size_t(D->nb) * 8, size_t(D->nb), cudaMemcpyDeviceToHost, D->copy));
    }
    const size_t nstat = D->h_nodes.size();
    // screen on the device; the per-node statistics come back only when a block failed
    CK(cudaMemsetAsync(D->d_bad, 0x7f, sizeof(int), st));
    CK(launch_pivot_screen(D->d_pivstat, D->d_chk, int(nstat), want_G ? 1 : 0, D->d_bad, st));
    CK(cudaMemcpyAsync(D->h_bad, D->d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (want_G) CK(cudaMemcpyAsync(D->h_norm, D->d_norm, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (!D->h_qr.empty())
      CK(cudaMemcpyAsync(D->h_qstat, D->d_qstat, 2 * D->h_qr.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    const auto hs0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st));
    if (std::getenv("DTN_TRACE_BUILD"))
      std::fprintf(stderr, "[build] wait for the device %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hs0).count());
    if (opts->export_S) CK(cudaStreamSynchronize(D->copy));
    CK(cudaGetLastError());
    // singular blocks, first failing node in build order (dense_nd.cpp:93-96, 175-180)
    const Plan& P = D->P;
    const bool any_bad = *D->h_bad != 0x7f7f7f7f;
    if (any_bad) CK(cudaMemcpy(D->h_pivstat, D->d_pivstat, 2 * nstat * sizeof(double), cudaMemcpyDeviceToHost));
    if (any_bad)
      for (const Wave& wv : P.waves)
      for (const auto* lst : {&wv.micro, &wv.small, &wv.blocked})
        for (int id : *lst) {
          const Node& nd = P.nodes[id];
          if (nd.ni > 0 && !pivots_ok(D->h_pivstat[2 * id], D->h_pivstat[2 * id + 1])) {
            if (std::getenv("DTN_DEBUG"))
              std::fprintf(stderr, "dtn: node %d kind %d ni %d nb %d total %d blocked %d pmin %g pmax %g\n", id,
                           int(nd.kind), nd.ni, nd.nb, nd.total, int(nd.blocked), D->h_pivstat[2 * id],
                           D->h_pivstat[2 * id + 1]);
            throw Singular(label_of(P, nd));
          }
        }
    auto* op = new dtn_op;
    op->ctx = ctx;
    op->plan = D;
    op->nb = D->nb;
    op->has_G = want_G;
    if (want_G) {
      const int r = D->root_lu_node;
      if (any_bad && !pivots_ok(D->h_pivstat[2 * r], D->h_pivstat[2 * r + 1])) {
        delete op;
        throw Singular("root Schur complement is singular [root]");
      }
      double n1[2];
      std::memcpy(n1, D->h_norm, sizeof(n1));
      op->cond = n1[0] * n1[1];
    }
    // timings
    auto ms = [](cudaEvent_t a, cudaEvent_t b) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, a, b) != cudaSuccess) {
        (void)cudaGetLastError();  // not a sticky error: do not poison later launches
        return -1.0;
      }
      return double(t);
    };
    dtn_build_stats& s = op->stats;
    const bool graph_run = !profile && use_graphs() && !comm;
    s.build_ms = ms(D->ev_start, D->ev_end);
    s.inverse_ms = graph_run ? 0.0 : ms(D->ev_root, D->ev_end);
    s.merge_flops = P.merge_flops;
    s.leaf_flops = P.micro_flops;
    s.inverse_flops = want_G ? 2.0 * double(D->nb) * D->nb * D->nb : 0.0;
    s.waves = int(P.waves.size());
    s.launches = D->launches;
    s.arena_bytes = double(P.arena_peak_bytes);
    s.arena_sum_bytes = double(P.arena_sum_bytes);
    std::vector<dtn_level_stats> lv(P.depth + 1);
    for (int l = 0; l <= P.depth; ++l) {
      lv[l].level = l;
      lv[l].boxes = int(P.levels[l].size());
      for (int id : P.levels[l]) {
        lv[l].max_boundary = std::max<int64_t>(lv[l].max_boundary, perimeter_size(P.boxes[id].r));
        const int v = P.boxes[id].node;
        if (v < 0 || !P.active[v]) continue;
        const Node& nd = P.nodes[v];
        lv[l].bytes += uint64_t(8) * uint64_t(nd.nb) * uint64_t(nd.nb) +
                       (nd.factors ? uint64_t(8) * uint64_t(nd.ell) * uint64_t(2 * nd.jn + 2 * nd.nb) : 0);
      }
    }
    // structured merges: numerical ranks and the range-finder check per level
    s.exec_flops = 0.0;
    for (const WaveLaunch& W : D->wl) s.exec_flops += W.sm_flops + W.cp_flops + W.fin_flops;
    for (const Node& nd : P.nodes)
      if (nd.smerge) {
        ++s.structured_merges;
        s.exec_flops += merge_flop_count(nd.ni, nd.sys_nb) - 2.0 * nd.sys_nb * double(nd.sys_nb) * nd.ni;
      }
    for (size_t q = 0; q < D->h_qr.size(); ++q) {
      const Node& nd = P.nodes[size_t(D->qr_node[q])];
      const int rank = int(D->h_qstat[2 * q]);
      s.max_rank = std::max(s.max_rank, rank);
      s.sketch_tail = std::max(s.sketch_tail, D->h_qstat[2 * q + 1]);
      // (a W/E half counts with its merge_four's level, a reference leaf with the leaves)
      const int l = std::min(std::max(nd.label_level >= 0 ? nd.label_level : P.depth, 0), P.depth);
      lv[size_t(l)].max_rank = std::max<int64_t>(lv[size_t(l)].max_rank, rank);
    }
    cudaEvent_t prev = D->ev_start;
    for (size_t w = 0; w < D->wl.size(); ++w) {
      const double t = graph_run ? 0.0 : ms(prev, D->ev_wave[w]);
      prev = D->ev_wave[w];
      const int l = D->wl[w].level;
      if (l < 0) {
        s.leaf_ms += t;
        lv[P.depth].seconds += t * 1e-3;
        lv[P.depth].flops += D->wl[w].flops;
      } else {
        s.merge_ms += t;
        lv[l].seconds += t * 1e-3;
        lv[l].flops += D->wl[w].flops;
      }
    }
    op->levels = std::move(lv);
    if (prof) {
      op->kstats.assign(K_COUNT, dtn_kernel_stats{});
      for (int k = 0; k < K_COUNT; ++k) std::snprintf(op->kstats[k].name, sizeof(op->kstats[k].name), "%s", kclass_name(k));
      // DTN_PROF_DUMP=1: the launch timeline on stderr (wave, class, start, duration)
      const char* dump = std::getenv("DTN_PROF_DUMP");
      if (dump && dump[0] == '1') {
        std::fprintf(stderr, "prof panel fallbacks %u small fallbacks %u\n", panel_fallbacks_read_reset(),
                     small_fallbacks_read_reset());
        // per wave: blocked merges whose panels needed row interchanges
        for (size_t w = 0; w < P.waves.size(); ++w) {
          int cnt = 0, tot = 0;
          for (int id : P.waves[w].blocked) {
            const Node& nd = P.nodes[id];
            int flag = 0;
            cudaMemcpy(&flag, D->d_piv + nd.piv_off + align_up(std::max(nd.ni, 1), 4) + 256, sizeof(int),
                       cudaMemcpyDeviceToHost);
            cnt += flag;
            ++tot;
          }
          if (tot) std::fprintf(stderr, "prof wave %zu pivoting panels %d in %d merges\n", w, cnt, tot);
        }
      }
      if (dump && dump[0] == '1' && !prof->recs.empty())
        for (auto& r : prof->recs)
          std::fprintf(stderr, "prof wave %3d %-14s start %9.4f ms dur %8.4f ms gflop %8.4f\n", r.wave,
                       kclass_name(r.kclass), ms(prof->recs.front().a, r.a), ms(r.a, r.b), r.flops * 1e-9);
      for (auto& r : prof->recs) {
        dtn_kernel_stats& ks = op->kstats[r.kclass];
        const double t = ms(r.a, r.b);
        ks.launches += 1;
        ks.ms += t;
        ks.max_ms = std::max(ks.max_ms, t);
        ks.flops += r.flops;
        ks.bytes += r.bytes;
      }
    }
    D->busy = true;
    *out = op;
  });
}

// Range-finder acceptance: the probe residual |(I - Q Q^T) S[J, K] w| relative to the box
// operator's scale must be <= factor * eps (DTN_RANK_TOL, default 1: the truncation of a
// factor then perturbs S by ~eps |S|, the scale of the reference's eps sigma_max cuts).
double rank_tol_factor() {
  static const double v = [] {
    const char* e = std::getenv("DTN_RANK_TOL");
    return e ? std::atof(e) : 1.0;
  }();
  return v;
}

// Step of a rank raise: ell / DTN_RANK_RAISE (at least 16).
int rank_raise_div() {
  static const int v = [] {
    const char* e = std::getenv("DTN_RANK_RAISE");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  return v;
}

int rank_raise_fine() {  // DTN_RANK_RAISE_FINE=0: always the full step
  static const int v = [] {
    const char* e = std::getenv("DTN_RANK_RAISE_FINE");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// Factor ranks that failed the range-finder check of a structured build (tail of the
// sketch's R diagonal above tol): raise them by ell / DTN_RANK_RAISE (at least 16), per
// J edge size.
bool raise_ranks(const dtn_op* op, double tol, std::vector<std::pair<int, int>>& over) {
  const PlanDev& D = *op->plan;
  bool raised = false;
  for (size_t q = 0; q < D.h_qr.size(); ++q) {
    if (!(D.h_qstat[2 * q + 1] > tol)) continue;
    const Node& nd = D.P.nodes[size_t(D.qr_node[q])];
    if (nd.ell >= nd.jn) continue;  // already exact
    // far from resolved (probe residual > 30 tol): ell / DTN_RANK_RAISE (at least 16); close to it
    // (the residual falls geometrically with the rank): half that step (at least 8), so that the
    // learned rank ends near the numerical one instead of a full step above it
    const bool far = !(D.h_qstat[2 * q + 1] <= 30.0 * tol) || rank_raise_fine() == 0;
    const int step = far ? std::max(16, nd.ell / rank_raise_div()) : std::max(8, nd.ell / (2 * rank_raise_div()));
    const int want = std::min({nd.jn, 252, int(align_up(nd.ell + step, 8))});
    if (want <= nd.ell) continue;  // at the cap
    auto it = std::find_if(over.begin(), over.end(), [&](const auto& e) { return e.first == nd.jn; });
    if (it == over.end()) {
      over.push_back({nd.jn, want});
      raised = true;
    } else if (it->second < want) {
      it->second = want;
      raised = true;
    }
  }
  return raised;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

int build_adaptive(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, dtn_op** out, int world = 1,
                   int wrank = -1, void* comm = nullptr) {
  if (!ctx || !opts || opts->engine != 1) return build_impl(ctx, prob, opts, {}, out, world, wrank, comm);
  // structured merges: the factor ranks adapt to the operator. A build whose sketches
  // did not resolve a factor to eps (the probe residual relative to the box operator's
  // scale, cf. lowrank_from_dense's eps sigma_max cut, lowrank.cpp:27-36) is repeated
  // with those ranks raised; the learned ranks are kept in the context for later builds
  // of the same problem family.
  const double eps = opts->epsilon > 0.0 ? opts->epsilon : 1e-10;
  char fam[256];
  std::snprintf(fam, sizeof(fam), "%d/%d/%d/%lld/%d/%d/%d/%d/%g", prob ? prob->n : 0, opts->n_leaf, opts->leaf_side,
                (long long)opts->crossover, opts->nshards, opts->shard, opts->rank_base, opts->rank_step, eps);
  std::vector<std::pair<int, int>> over;
  {
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    auto it = ctx->learned_ranks.find(fam);
    if (it != ctx->learned_ranks.end()) over = it->second;
  }
  for (int attempt = 0;; ++attempt) {
    dtn_op* op = nullptr;
    const int rc = build_impl(ctx, prob, opts, over, &op, world, wrank, comm);
    if (rc != DTN_OK) return rc;
    std::vector<std::pair<int, int>> next = over;
    if (attempt < 8 && raise_ranks(op, rank_tol_factor() * eps, next)) {
      PlanDev* stale = op->plan;
      dtn_gpu_free(op);
      {  // the failed attempt's plan (arena, graph) is not reused: drop it
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        auto& pl = ctx->plans;
        pl.erase(std::remove_if(pl.begin(), pl.end(), [&](const auto& p) { return p.get() == stale; }), pl.end());
      }
      over = std::move(next);
      std::lock_guard<std::recursive_mutex> lk(ctx->mu);
      ctx->learned_ranks[fam] = over;
      continue;
    }
    op->stats.rank_attempts = attempt + 1;
    *out = op;
    return DTN_OK;
  }
}

// Collective build over `world` GPUs (one process per GPU, opts->shard == -2):
// rank r builds shard r's subtree (no communication), the shard S blocks are gathered to
// every rank (ncclAllGather), then every rank runs the top of the tree with its blocked
// merges column-sharded -- interface LU redundant, this rank's chunk of the boundary
// columns' substitutions and Schur GEMM, ncclAllGather of the chunks after each wave --
// so the root S (and G) ends up on every rank. opts->shard == -3: the same split with
// every shard and every chunk computed on this device (no communication), which
// checks the partition on one GPU.
int build_collective(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, dtn_op** out) {
  const int N = opts->nshards;
  const bool real = opts->shard == -2;
  // -4 (loopback): -3's single-device split with every NCCL call of the real path issued on the
  // context's 1-rank communicator (in place: no data moves) -- exercises the dlopen'ed API, the
  // communicator and the collectives captured in the build graph on one GPU
  const bool loop = opts->shard == -4;
  std::vector<int64_t> nbs(static_cast<size_t>(N), 0);
  int rc = guarded(ctx, [&] {
    if (!prob || !out) throw std::invalid_argument("dtn_gpu_build: null argument");
    if (loop && (ctx->world != 1 || !ctx->comm))
      throw std::invalid_argument("collective loopback: the context needs a 1-rank communicator (dtn_gpu_create_rank)");
    if (real && (ctx->world != N || !ctx->comm))
      throw std::invalid_argument("collective build: nshards must equal the context's NCCL world (dtn_gpu_create_rank)");
    if (opts->nloads > 0) throw std::invalid_argument("dtn_gpu_build: body loads are not supported in sharded builds");
    int32_t rect[4];
    for (int r = 0; r < N; ++r) {
      const int e = dtn_gpu_shard_info(prob->n, opts->n_leaf, opts->leaf_side, N, r, rect, &nbs[size_t(r)]);
      if (e != DTN_OK) throw std::invalid_argument(dtn_gpu_last_error(nullptr));
    }
  });
  if (rc != DTN_OK) return rc;
  int64_t slot = 0;
  for (int64_t b : nbs) slot = std::max(slot, b * b);
  slot = align_up(slot, 32);
  rc = guarded(ctx, [&] {
    CK(cudaSetDevice(ctx->device));
    if (ctx->gather_cap < size_t(N) * size_t(slot)) {
      if (ctx->d_gather) cudaFree(ctx->d_gather);
      ctx->d_gather = nullptr;
      ctx->gather_cap = 0;
      CK(cudaMalloc(&ctx->d_gather, size_t(N) * size_t(slot) * 8));
      ctx->gather_cap = size_t(N) * size_t(slot);
    }
  });
  if (rc != DTN_OK) return rc;
  cudaStream_t st = ctx->stream;
  for (int r = 0; r < N; ++r) {
    if (real && r != ctx->rank) continue;
    dtn_opts os = *opts;
    os.shard = r;
    os.want_G = 0;
    os.export_S = nullptr;
    dtn_op* sop = nullptr;
    rc = build_adaptive(ctx, prob, &os, &sop);
    if (rc != DTN_OK) return rc;
    rc = guarded(ctx, [&] {
      const PlanDev& D = *sop->plan;
      CK(cudaMemcpy2DAsync(ctx->d_gather + size_t(r) * slot, size_t(nbs[size_t(r)]) * 8, D.d_S, size_t(D.lds) * 8,
                           size_t(nbs[size_t(r)]) * 8, size_t(nbs[size_t(r)]), cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
    });
    dtn_gpu_free(sop);
    if (rc != DTN_OK) return rc;
  }
  if (real || loop) {
    rc = guarded(ctx, [&] {
      nccl_check(nccl().AllGather(ctx->d_gather + size_t(ctx->rank) * slot, ctx->d_gather, size_t(slot), ncclDouble,
                                  ctx->comm, st),
                 "ncclAllGather (shard S)");
      CK(cudaStreamSynchronize(st));
    });
    if (rc != DTN_OK) return rc;
  }
  std::vector<const double*> ptrs(static_cast<size_t>(N), nullptr);
  for (int r = 0; r < N; ++r) ptrs[size_t(r)] = ctx->d_gather + size_t(r) * slot;
  dtn_problem pt = *prob;
  pt.shard_S = ptrs.data();
  pt.shard_S_on_device = 1;
  dtn_opts ot = *opts;
  ot.shard = -1;
  return build_adaptive(ctx, &pt, &ot, out, N, real ? ctx->rank : -1,
                        (real || loop) ? static_cast<void*>(ctx->comm) : nullptr);
}

}  // namespace

extern "C" {

int dtn_gpu_build(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, dtn_op** out) {
  if (ctx && opts && opts->nshards > 1 && (opts->shard == -2 || opts->shard == -3 || opts->shard == -4))
    return build_collective(ctx, prob, opts, out);
  return build_adaptive(ctx, prob, opts, out);
}

void dtn_gpu_free(dtn_op* op) {
  if (!op) return;
  if (op->plan) op->plan->busy = false;
  delete op;
}

int dtn_gpu_boundary(const dtn_op* op, int64_t* ids, int64_t* nb) {
  if (!op || !nb) return DTN_EINVAL;
  *nb = op->nb;
  if (ids) {
    const Plan& P = op->plan->P;
    std::vector<std::pair<int, int>> per;
    perimeter_ccw(P.nodes[P.root].r, per);
    const int side = P.n - 2;
    for (size_t i = 0; i < per.size(); ++i) ids[i] = int64_t(per[i].second - 1) * side + (per[i].first - 1);
  }
  return DTN_OK;
}

int dtn_gpu_export(const dtn_op* op, double* S, double* G, double* cond) {
  if (!op) return DTN_EINVAL;
  return guarded(op->ctx, [&] {
    CK(cudaSetDevice(op->ctx->device));
    const PlanDev& D = *op->plan;
    const size_t nb = size_t(op->nb);
    if (S) CK(cudaMemcpy2D(S, nb * 8, D.d_S, size_t(D.lds) * 8, nb * 8, nb, cudaMemcpyDeviceToHost));
    if (G) {
      if (!op->has_G) throw std::invalid_argument("dtn_gpu_export: G was not built (want_G = 0)");
      CK(cudaMemcpy2D(G, nb * 8, D.d_G, size_t(D.ldg) * 8, nb * 8, nb, cudaMemcpyDeviceToHost));
    }
    if (cond) *cond = op->cond;
  });
}

int dtn_gpu_export_device(const dtn_op* op, double* S, int64_t lds, double* G, int64_t ldg) {
  if (!op) return DTN_EINVAL;
  return guarded(op->ctx, [&] {
    CK(cudaSetDevice(op->ctx->device));
    const PlanDev& D = *op->plan;
    const size_t nb = size_t(op->nb);
    cudaStream_t st = op->ctx->stream;
    if (S) {
      if (lds < int64_t(nb)) throw std::invalid_argument("dtn_gpu_export_device: lds < nb");
      CK(cudaMemcpy2DAsync(S, size_t(lds) * 8, D.d_S, size_t(D.lds) * 8, nb * 8, nb, cudaMemcpyDeviceToDevice, st));
    }
    if (G) {
      if (!op->has_G) throw std::invalid_argument("dtn_gpu_export_device: G was not built (want_G = 0)");
      if (ldg < int64_t(nb)) throw std::invalid_argument("dtn_gpu_export_device: ldg < nb");
      CK(cudaMemcpy2DAsync(G, size_t(ldg) * 8, D.d_G, size_t(D.ldg) * 8, nb * 8, nb, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

int dtn_gpu_device_ptrs(const dtn_op* op, const double** S, const double** G, int64_t* ld) {
  if (!op) return DTN_EINVAL;
  if (S) *S = op->plan->d_S;
  if (G) *G = op->has_G ? op->plan->d_G : nullptr;
  if (ld) *ld = op->plan->lds;
  return DTN_OK;
}

int dtn_gpu_body_map(const dtn_op* op, double* F, int64_t ldf, int on_device) {
  if (!op) return DTN_EINVAL;
  dtn_ctx* ctx = op->ctx;
  return guarded(ctx, [&] {
    const PlanDev& D = *op->plan;
    const int nl = D.P.key.nloads;
    if (nl == 0) throw std::invalid_argument("dtn_gpu_body_map: the build had no body loads");
    if (!op->has_G) throw std::invalid_argument("dtn_gpu_body_map: body loads need G (want_G)");
    if (!F || ldf < op->nb) throw std::invalid_argument("dtn_gpu_body_map: bad output");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpy2DAsync(F, size_t(ldf) * 8, D.d_F, size_t(D.ldf) * 8, size_t(op->nb) * 8, size_t(nl),
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int dtn_gpu_root_rhs(const dtn_op* op, double* R, int64_t ldr, int on_device) {
  if (!op) return DTN_EINVAL;
  dtn_ctx* ctx = op->ctx;
  return guarded(ctx, [&] {
    const PlanDev& D = *op->plan;
    const int nl = D.P.key.nloads;
    if (nl == 0) throw std::invalid_argument("dtn_gpu_root_rhs: the build had no body loads");
    if (!R || ldr < op->nb) throw std::invalid_argument("dtn_gpu_root_rhs: bad output");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpy2DAsync(R, size_t(ldr) * 8, D.d_arena + D.rhs_root_off, size_t(D.rhs_root_ld) * 8,
                         size_t(op->nb) * 8, size_t(nl), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int dtn_gpu_ring_dtn(const dtn_op* op, const int64_t* adj, const double* coef, int64_t m, double h, double* T,
                     int64_t ldt, int on_device) {
  if (!op) return DTN_EINVAL;
  dtn_ctx* ctx = op->ctx;
  return guarded(ctx, [&] {
    const int nb = op->nb;
    if (!op->has_G) throw std::invalid_argument("dtn_gpu_ring_dtn: G was not built (want_G = 0)");
    if (m < 0 || m > (int64_t(1) << 30) || ldt < m || (m && (!adj || !coef || !T)) || !(h > 0.0))
      throw std::invalid_argument("dtn_gpu_ring_dtn: bad arguments");
    std::vector<int> a32(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) {
      if (adj[i] < 0 || adj[i] >= nb) throw std::invalid_argument("dtn_gpu_ring_dtn: adjacency outside the boundary");
      a32[size_t(i)] = int(adj[i]);
    }
    if (m == 0) return;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const PlanDev& D = *op->plan;
    int* d_adj = nullptr;
    double *d_coef = nullptr, *d_T = nullptr;
    CK(cudaMallocAsync(&d_adj, size_t(m) * sizeof(int), st));
    CK(cudaMallocAsync(&d_coef, size_t(m) * sizeof(double), st));
    CK(cudaMemcpyAsync(d_adj, a32.data(), size_t(m) * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_coef, coef, size_t(m) * sizeof(double), cudaMemcpyHostToDevice, st));
    double* out = T;
    int64_t ldo = ldt;
    if (!on_device) {
      CK(cudaMallocAsync(&d_T, size_t(m) * size_t(m) * sizeof(double), st));
      out = d_T;
      ldo = m;
    }
    CK(launch_ring_dtn(D.d_G, D.ldg, d_adj, d_coef, int(m), h, out, ldo, st));
    if (!on_device)
      CK(cudaMemcpy2DAsync(T, size_t(ldt) * 8, d_T, size_t(m) * 8, size_t(m) * 8, size_t(m), cudaMemcpyDeviceToHost,
                           st));
    CK(cudaFreeAsync(d_adj, st));
    CK(cudaFreeAsync(d_coef, st));
    if (d_T) CK(cudaFreeAsync(d_T, st));
    CK(cudaStreamSynchronize(st));
  });
}

int dtn_gpu_apply(const dtn_op* op, int which, const double* X, int64_t ldx, int64_t batch, double* Y, int64_t ldy,
                  int on_device) {
  if (!op) return DTN_EINVAL;
  dtn_ctx* ctx = op->ctx;
  return guarded(ctx, [&] {
    const int nb = op->nb;
    if (which != 0 && which != 1) throw std::invalid_argument("dtn_gpu_apply: which must be 0 (G) or 1 (S)");
    if (which == 0 && !op->has_G) throw std::invalid_argument("apply_dtn: G was not built (want_G = 0)");
    if (batch < 0 || ldx < nb || ldy < nb || (!X && batch) || (!Y && batch))
      throw std::invalid_argument("apply: boundary vector size mismatch");
    if (batch == 0) return;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const PlanDev& D = *op->plan;
    const double* A = which == 0 ? D.d_G : D.d_S;
    const int lda = which == 0 ? D.ldg : D.lds;
    const bool aligned = on_device && (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (ldx % 2 == 0) &&
                         (reinterpret_cast<uintptr_t>(Y) % 16 == 0) && (ldy % 2 == 0);
    const double* dX = X;
    double* dY = Y;
    int64_t ldX = ldx, ldY = ldy;
    if (!aligned) {
      const int64_t ldp = align_up(nb, 2);
      const size_t need = size_t(ldp) * size_t(batch);
      if (need > ctx->stage_cap) {
        if (ctx->d_x) cudaFree(ctx->d_x);
        if (ctx->d_y) cudaFree(ctx->d_y);
        ctx->d_x = ctx->d_y = nullptr;
        ctx->stage_cap = 0;
        CK(cudaMalloc(&ctx->d_x, need * 8));
        CK(cudaMalloc(&ctx->d_y, need * 8));
        ctx->stage_cap = need;
      }
      CK(cudaMemcpy2DAsync(ctx->d_x, size_t(ldp) * 8, X, size_t(ldx) * 8, size_t(nb) * 8, size_t(batch),
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
      dX = ctx->d_x;
      dY = ctx->d_y;
      ldX = ldY = ldp;
    }
    if (batch <= 32) {  // HBM-bound stream over the operator: split-K skinny product
      const size_t wd = skinny_work_doubles(nb, nb, int(batch));
      if (wd > ctx->skinny_cap) {
        if (ctx->d_skinny) pool_free(ctx->d_skinny);
        ctx->d_skinny = static_cast<double*>(pool_alloc(wd * 8));
        ctx->skinny_cap = wd;
      }
      CK(launch_skinny_gemm(A, lda, dX, int(ldX), dY, int(ldY), nb, nb, int(batch), ctx->d_skinny, st));
    } else {
      GemmDesc d{A, dX, dY, nb, int(batch), nb, lda, int(ldX), int(ldY)};
      alignas(64) unsigned char img[512] = {0};  // descriptor, and its A / B tensor maps at byte 256
      std::memcpy(img, &d, sizeof(d));
      const int tiles = gemm_tiles(nb, int(batch));
      const bool tma = tiles >= gemm_tma_min_tiles() && tma_encode_one(d, img + 256);
      CK(cudaMemcpyAsync(ctx->d_desc, img, tma ? 512 : sizeof(d), cudaMemcpyHostToDevice, st));
      if (tma)
        CK(launch_gemm_tma(ctx->d_desc, reinterpret_cast<const unsigned char*>(ctx->d_desc) + 256, 1, tiles, 1.0, 0.0, st));
      else
        CK(launch_gemm_desc(ctx->d_desc, 1, tiles, nb, 1.0, 0.0, st, true));
    }
    if (!aligned)
      CK(cudaMemcpy2DAsync(Y, size_t(ldy) * 8, dY, size_t(ldY) * 8, size_t(nb) * 8, size_t(batch),
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int dtn_gpu_num_boxes(const dtn_op* op, int32_t* count, int32_t* depth) {
  if (!op) return DTN_EINVAL;
  if (count) *count = int32_t(op->plan->P.boxes.size());
  if (depth) *depth = op->plan->P.depth;
  return DTN_OK;
}

int dtn_gpu_box_info(const dtn_op* op, int32_t box, int32_t* info) {
  if (!op || !info || box < 0 || box >= int32_t(op->plan->P.boxes.size())) return DTN_EINVAL;
  const RefBox& b = op->plan->P.boxes[box];
  const int32_t v[11] = {b.level, b.parent, b.r.x0, b.r.x1, b.r.y0, b.r.y1, perimeter_size(b.r),
                         b.children[0], b.children[1], b.children[2], b.children[3]};
  std::copy(v, v + 11, info);
  return DTN_OK;
}

int dtn_gpu_box_schur(const dtn_op* op, int32_t box, double* S) {
  if (!op || box < 0 || box >= int32_t(op->plan->P.boxes.size())) return DTN_EINVAL;
  return guarded(op->ctx, [&] {
    const PlanDev& D = *op->plan;
    const int node = D.P.boxes[box].node;
    if (node < 0) throw std::invalid_argument("dtn_gpu_box_schur: empty box");
    if (!D.P.active[node]) throw std::invalid_argument("dtn_gpu_box_schur: box not computed by this (sharded) build");
    if (!D.P.key.keep && node != D.P.root)
      throw std::invalid_argument("dtn_gpu_box_schur: box storage was reused (build with opts.keep_boxes = 1)");
    const Node& nd = D.P.nodes[node];
    CK(cudaSetDevice(op->ctx->device));
    CK(cudaMemcpy2D(S, size_t(nd.nb) * 8, D.d_arena + nd.s_off, size_t(nd.ld) * 8, size_t(nd.nb) * 8, nd.nb,
                    cudaMemcpyDeviceToHost));
  });
}

int dtn_gpu_level_stats(const dtn_op* op, dtn_level_stats* out, int32_t max, int32_t* count) {
  if (!op || !count) return DTN_EINVAL;
  *count = int32_t(op->levels.size());
  if (out)
    for (int32_t i = 0; i < std::min<int32_t>(max, *count); ++i) out[i] = op->levels[i];
  return DTN_OK;
}

int dtn_gpu_kernel_stats(const dtn_op* op, dtn_kernel_stats* out, int32_t max, int32_t* count) {
  if (!op || !count) return DTN_EINVAL;
  *count = int32_t(op->kstats.size());
  if (out)
    for (int32_t i = 0; i < std::min<int32_t>(max, *count); ++i) out[i] = op->kstats[i];
  return DTN_OK;
}

int dtn_gpu_build_stats(const dtn_op* op, dtn_build_stats* out) {
  if (!op || !out) return DTN_EINVAL;
  *out = op->stats;
  return DTN_OK;
}

int dtn_gpu_shard_info(int32_t n, int32_t n_leaf, int32_t leaf_side, int32_t nshards, int32_t shard, int32_t* rect,
                       int64_t* nb) {
  return guarded(nullptr, [&] {
    PlanKey key;
    key.n = n;
    key.n_leaf = n_leaf;
    key.leaf_side = leaf_side;
    key.micro_max = kDefaultMicro;
    key.small_max = kSmallMax;
    const Plan P = make_plan(key);
    const std::vector<int> sh = shard_nodes(P, nshards);
    if (shard < 0 || shard >= int(sh.size())) throw std::invalid_argument("shards: shard index out of range");
    const Node& nd = P.nodes[sh[shard]];
    if (rect) {
      rect[0] = nd.r.x0;
      rect[1] = nd.r.x1;
      rect[2] = nd.r.y0;
      rect[3] = nd.r.y1;
    }
    if (nb) *nb = nd.nb;
  });
}

// Work per rank of a collective build (host only): shard r's subtree, plus the top of
// the tree with every column-sharded merge's interface LU redundant and its boundary
// columns' substitutions (2 ni^2 per column) and Schur GEMM (2 nb ni per column) split
// by chunk, small merges redundant, and (want_G) the root inverse as a redundant LU of
// S plus this rank's chunk of the substitutions (2 nb^2 per column).
int dtn_gpu_collective_flops(int32_t n, int32_t n_leaf, int32_t leaf_side, int32_t nranks, int32_t want_G,
                             double* per_rank, double* single_gpu) {
  return guarded(nullptr, [&] {
    if (nranks < 2 || !per_rank) throw std::invalid_argument("dtn_gpu_collective_flops: bad arguments");
    PlanKey key;
    key.n = n;
    key.n_leaf = n_leaf;
    key.leaf_side = leaf_side;
    key.micro_max = kDefaultMicro;
    key.small_max = kSmallMax;
    const Plan full = make_plan(key);
    const int nb = full.nodes[full.root].nb;
    if (single_gpu) *single_gpu = full.merge_flops + full.micro_flops + (want_G ? 2.0 * nb * double(nb) * nb : 0.0);
    for (int r = 0; r < nranks; ++r) {
      PlanKey ks = key;
      ks.nshards = nranks;
      ks.shard = r;
      const Plan sp = make_plan(ks);
      double f = sp.merge_flops + sp.micro_flops;
      PlanKey kt = key;
      kt.nshards = nranks;
      kt.shard = -1;
      kt.world = nranks;
      kt.wrank = r;
      const Plan tp = make_plan(kt);
      for (size_t v = 0; v < tp.nodes.size(); ++v) {
        const Node& nd = tp.nodes[v];
        if (!tp.active[v] || nd.kind != NodeKind::merge) continue;
        if (!nd.colshard) {
          f += merge_flop_count(nd.ni, nd.nb);
          continue;
        }
        const int c0 = r * nd.cw, c1 = std::min(nd.nb, c0 + nd.cw);
        const double cols = std::max(0, c1 - c0);
        f += (2.0 / 3.0) * nd.ni * double(nd.ni) * nd.ni + cols * (2.0 * nd.ni * double(nd.ni) + 2.0 * nd.nb * double(nd.ni));
      }
      if (want_G) {
        const int cw = (nb + nranks - 1) / nranks, c0 = r * cw, c1 = std::min(nb, c0 + cw);
        f += (2.0 / 3.0) * nb * double(nb) * nb + 2.0 * nb * double(nb) * std::max(0, c1 - c0);
      }
      per_rank[r] = f;
    }
  });
}

// Test hook: blocked partial LU of one dense n x n matrix with the engine's
// panel / rowpanel / trailing kernels (pivots among the first ni rows;
// ni == n is a full LU with left swaps, as for the root inverse).
int dtn_debug_partial_lu(int32_t n, int32_t ni, const double* A, double* out, int32_t* ipiv, double* pivstat) {
  return guarded(nullptr, [&] {
    if (n <= 0 || ni <= 0 || ni > n) throw std::invalid_argument("dtn_debug_partial_lu: bad sizes");
    CK(gemm_init());
    CK(gemm_tma_init());
    CK(fused_init());
    CK(blocked_init());
    const int ld = int(align_up(n, 8));
    NodeDev nd{};
    nd.kind = 2;
    nd.nb = n - ni;
    nd.ni = ni;
    nd.total = n;
    nd.ncols = n;
    nd.a = nd.b = -1;
    nd.ld = nd.ldm = ld;
    NodeDev* d_node = dalloc<NodeDev>(1);
    int* d_list = dalloc<int>(1);
    double* d_a = dalloc<double>(size_t(ld) * n);
    int* d_piv = dalloc<int>(size_t(align_up(n, 4) + 260));
    double* d_ps = dalloc<double>(2);
    int zero = 0;
    CK(cudaMemcpy(d_node, &nd, sizeof(nd), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_list, &zero, sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy2D(d_a, size_t(ld) * 8, A, size_t(n) * 8, size_t(n) * 8, n, cudaMemcpyHostToDevice));
    KernelArgs a{d_node, nullptr, nullptr, 0, 0, d_a, d_piv, d_ps};
    // DTN_DEBUG_LU_FUSED=1 (full LU only): the fused look-ahead sequence of
    // the root LU, serialised on one stream
    const char* fe = std::getenv("DTN_DEBUG_LU_FUSED");
    const bool fused = ni == n && fe && fe[0] == '1';
    for (int k0 = 0; k0 < ni; k0 += 32) {
      CK(launch_panel(a, d_list, 1, ni - k0, k0, 32, 0, fused));
      CK(launch_rowpanel(a, d_list, 1, n, n - ni, k0, 32, ni == n, 0, fused));
      CK(launch_trailing_update(a, d_list, 1, n, k0, 32, fused ? -1 : 0, 1 << 30, 0, fused ? n : 0));
    }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy2D(out, size_t(n) * 8, d_a, size_t(ld) * 8, size_t(n) * 8, n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ipiv, d_piv, size_t(ni) * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pivstat, d_ps, 2 * sizeof(double), cudaMemcpyDeviceToHost));
    for (void* p : std::initializer_list<void*>{d_node, d_list, d_a, d_piv, d_ps}) cudaFree(p);
  });
}

// Diagnostic: phase clocks of the fused merge kernel (3 size classes x 8 slots)
int dtn_debug_fused_clocks(int64_t* out24) {
  return guarded(nullptr, [&] {
    cudaDeviceSynchronize();
    fused_clocks_read(reinterpret_cast<long long*>(out24));
  });
}

// Test hook: C = alpha A B + beta C (host column-major operands, tight leading dimensions
// rounded up to even) through the engine's GEMM dispatch; path 0 = cp.async kernels,
// 1 = the TMA-staged kernel (k_tma.cu; fails if the tensor maps cannot be encoded).
int dtn_debug_gemm(int32_t m, int32_t n, int32_t k, const double* A, const double* B, double* Cio, double alpha,
                   double beta, int32_t path) {
  return guarded(nullptr, [&] {
    if (m <= 0 || n <= 0 || k <= 0 || !A || !B || !Cio) throw std::invalid_argument("dtn_debug_gemm: bad arguments");
    CK(gemm_init());
    CK(gemm_tma_init());
    CK(fused_init());
    const int lda = int(align_up(m, 2)), ldb = int(align_up(k, 2)), ldc = lda;
    double *dA = nullptr, *dB = nullptr, *dC = nullptr;
    unsigned char* dd = nullptr;
    CK(cudaMalloc(&dA, size_t(lda) * k * 8));
    CK(cudaMalloc(&dB, size_t(ldb) * n * 8));
    CK(cudaMalloc(&dC, size_t(ldc) * n * 8));
    CK(cudaMalloc(&dd, 512));
    CK(cudaMemcpy2D(dA, size_t(lda) * 8, A, size_t(m) * 8, size_t(m) * 8, size_t(k), cudaMemcpyHostToDevice));
    CK(cudaMemcpy2D(dB, size_t(ldb) * 8, B, size_t(k) * 8, size_t(k) * 8, size_t(n), cudaMemcpyHostToDevice));
    CK(cudaMemcpy2D(dC, size_t(ldc) * 8, Cio, size_t(m) * 8, size_t(m) * 8, size_t(n), cudaMemcpyHostToDevice));
    GemmDesc d{dA, dB, dC, m, n, k, lda, ldb, ldc};
    alignas(64) unsigned char img[512] = {0};
    std::memcpy(img, &d, sizeof(d));
    const bool tma = path == 1;
    bool enc = true;
    if (tma) enc = tma_encode_one(d, img + 256);
    cudaError_t e = cudaSuccess;
    if (enc) {
      CK(cudaMemcpy(dd, img, 512, cudaMemcpyHostToDevice));
      const GemmDesc* gd = reinterpret_cast<const GemmDesc*>(dd);
      e = tma ? launch_gemm_tma(gd, dd + 256, 1, gemm_tiles(m, n), alpha, beta, 0)
              : launch_gemm_desc(gd, 1, gemm_tiles(m, n), k, alpha, beta, 0, true);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e == cudaSuccess)
        e = cudaMemcpy2D(Cio, size_t(m) * 8, dC, size_t(ldc) * 8, size_t(m) * 8, size_t(n), cudaMemcpyDeviceToHost);
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    cudaFree(dd);
    if (!enc) throw std::runtime_error("dtn_debug_gemm: no tensor maps for this shape (TMA unavailable or disabled)");
    CK(e);
  });
}

// discretize, continuum branch (grid.cpp:130-144): paper's 1/h convection scaling
int dtn_discretize_continuum(int32_t n, const double* b, const double* c, const double* d, double* st) {
  if (n < 4 || !st) return DTN_EINVAL;
  const int64_t s = n - 2, nu = s * s;
  const double h = 1.0 / (n - 1), ih2 = 1.0 / (h * h), ih = 1.0 / h;
  for (int64_t k = 0; k < nu; ++k) {
    const double bv = b ? b[k] : 0.0, cv = c ? c[k] : 0.0, dv = d ? d[k] : 0.0;
    if (!std::isfinite(bv) || !std::isfinite(cv) || !std::isfinite(dv)) return DTN_EINVAL;
    st[k] = 4.0 * ih2 + dv;
    st[nu + k] = -ih2 + bv * ih;
    st[2 * nu + k] = -ih2 - bv * ih;
    st[3 * nu + k] = -ih2 + cv * ih;
    st[4 * nu + k] = -ih2 - cv * ih;
  }
  return DTN_OK;
}

// discretize, network branch (grid.cpp:82-92, 145-150): std::mt19937_64,
// u = (rng() >> 11) * 2^-53, horizontal links row-major then vertical links
int dtn_discretize_network(int32_t n, double lo, double hi, uint64_t seed, double* st) {
  if (n < 4 || !st) return DTN_EINVAL;
  const int64_t s = n - 2, nu = s * s;
  std::vector<double> sigma(size_t(2) * n * (n - 1));
  std::mt19937_64 rng(seed);
  for (auto& v : sigma) v = lo + (hi - lo) * (double(rng() >> 11) * 0x1.0p-53);
  auto sh = [&](int x, int y) { return sigma[size_t(y) * (n - 1) + x]; };
  auto sv = [&](int x, int y) { return sigma[size_t(n) * (n - 1) + size_t(y) * n + x]; };
  for (int y = 1; y <= n - 2; ++y)
    for (int x = 1; x <= n - 2; ++x) {
      const int64_t k = int64_t(y - 1) * s + (x - 1);
      const double se = sh(x, y), sw = sh(x - 1, y), sn = sv(x, y), ss = sv(x, y - 1);
      st[k] = se + sw + sn + ss;
      st[nu + k] = -se;
      st[2 * nu + k] = -sw;
      st[3 * nu + k] = -sn;
      st[4 * nu + k] = -ss;
    }
  return DTN_OK;
}

// ---- HBS (compressed) operators: compress (hbs.cpp:61-178), apply
// (hbs.cpp:187-232), DTNHBS01 (hbs.cpp:422-519); see csrc/hbs.cu
int dtn_gpu_hbs_compress(dtn_ctx* ctx, const double* H, int64_t M, int64_t ldh, int on_device, double eps,
                         int64_t leaf_cap, dtn_hbs** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (!H || M < 1 || ldh < M) throw std::invalid_argument("compress: matrix/tree size mismatch");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const double* dH = H;
    double* tmp = nullptr;
    int64_t ld = ldh;
    if (!on_device) {
      CK(cudaMalloc(&tmp, size_t(M) * M * 8));
      CK(cudaMemcpy2DAsync(tmp, size_t(M) * 8, H, size_t(ldh) * 8, size_t(M) * 8, size_t(M), cudaMemcpyHostToDevice,
                           st));
      dH = tmp;
      ld = M;
    }
    std::unique_ptr<HbsDev> h;
    try {
      h = hbs_compress(dH, ld, M, eps, leaf_cap, st);
    } catch (...) {
      if (tmp) cudaFree(tmp);
      throw;
    }
    if (tmp) cudaFree(tmp);
    auto* r = new dtn_hbs;
    r->ctx = ctx;
    r->h = std::move(h);
    *out = r;
  });
}

int dtn_gpu_hbs_compress_op(const dtn_op* op, int which, double eps, int64_t leaf_cap, dtn_hbs** out) {
  if (!op || !out) return DTN_EINVAL;
  dtn_ctx* ctx = op->ctx;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (which != 0 && which != 1) throw std::invalid_argument("compress: which must be 0 (G) or 1 (S)");
    if (which == 0 && !op->has_G) throw std::invalid_argument("compress: G was not built (want_G = 0)");
    CK(cudaSetDevice(ctx->device));
    const PlanDev& D = *op->plan;
    auto h = hbs_compress(which == 0 ? D.d_G : D.d_S, which == 0 ? D.ldg : D.lds, op->nb, eps, leaf_cap, ctx->stream);
    auto* r = new dtn_hbs;
    r->ctx = ctx;
    r->h = std::move(h);
    *out = r;
  });
}

void dtn_gpu_hbs_free(dtn_hbs* h) {
  if (!h) return;
  if (h->ctx) cudaSetDevice(h->ctx->device);
  delete h;
}

int dtn_gpu_hbs_info(const dtn_hbs* h, int64_t* M, int64_t* num_nodes, int32_t* depth, int64_t* max_rank,
                     uint64_t* payload_bytes) {
  if (!h || !h->h) return DTN_EINVAL;
  const HbsDev& H = *h->h;
  if (M) *M = H.M;
  if (num_nodes) *num_nodes = int64_t(H.nodes.size());
  if (depth) *depth = H.depth;
  if (max_rank) *max_rank = H.max_rank();
  if (payload_bytes) *payload_bytes = H.payload_bytes();
  return DTN_OK;
}

int dtn_gpu_hbs_tree(const dtn_hbs* h, int64_t* nodes, int64_t* ranks) {
  if (!h || !h->h) return DTN_EINVAL;
  const HbsDev& H = *h->h;
  for (size_t t = 0; t < H.nodes.size(); ++t) {
    const auto& n = H.nodes[t];
    if (nodes) {
      int64_t* o = nodes + 6 * t;
      o[0] = n.begin;
      o[1] = n.end;
      o[2] = n.left;
      o[3] = n.right;
      o[4] = n.parent;
      o[5] = n.level;
    }
    if (ranks) ranks[t] = t == 0 ? 0 : H.rank[t];
  }
  return DTN_OK;
}

int dtn_gpu_hbs_factor(const dtn_hbs* h, int32_t node, int32_t which, double* out, int64_t* rows, int64_t* cols) {
  if (!h || !h->h) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    const HbsDev& H = *h->h;
    if (node < 0 || node >= int32_t(H.nodes.size())) throw std::invalid_argument("hbs_factor: no such node");
    const bool leaf = H.is_leaf(node);
    const double* src = nullptr;
    int64_t r = 0, c = 0;
    switch (which) {
      case 0:  // D (leaves)
        if (!leaf) throw std::invalid_argument("hbs_factor: D exists on leaves only");
        src = H.D[node];
        r = c = H.node_size(node);
        break;
      case 1:
      case 2:  // U, V (non-root)
        if (node == 0) throw std::invalid_argument("hbs_factor: the root has no U/V");
        src = which == 1 ? H.U[node] : H.V[node];
        r = H.rows[node];
        c = H.rank[node];
        break;
      case 3:  // B (parents)
        if (leaf) throw std::invalid_argument("hbs_factor: B exists on parents only");
        src = H.B[node];
        r = c = H.rows[node];
        break;
      default:
        throw std::invalid_argument("hbs_factor: which must be 0 (D), 1 (U), 2 (V) or 3 (B)");
    }
    if (rows) *rows = r;
    if (cols) *cols = c;
    if (out && r > 0 && c > 0) {
      CK(cudaSetDevice(ctx->device));
      CK(cudaMemcpy2D(out, size_t(r) * 8, src, size_t(H.ld(node)) * 8, size_t(r) * 8, size_t(c),
                      cudaMemcpyDeviceToHost));
    }
  });
}

int dtn_gpu_hbs_apply(const dtn_hbs* h, const double* X, int64_t ldx, int64_t nrhs, double* Y, int64_t ldy,
                      int on_device) {
  if (!h || !h->h) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    HbsDev& H = *h->h;
    const int64_t M = H.M;
    if (nrhs < 0 || ldx < M || ldy < M || (!X && nrhs) || (!Y && nrhs))
      throw std::invalid_argument("apply: dimension mismatch");
    if (nrhs == 0) return;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    if (on_device) {
      hbs_apply(H, X, ldx, nrhs, Y, ldy, st);
    } else {
      const size_t need = size_t(M) * size_t(nrhs);
      if (need > ctx->stage_cap) {
        if (ctx->d_x) cudaFree(ctx->d_x);
        if (ctx->d_y) cudaFree(ctx->d_y);
        ctx->d_x = ctx->d_y = nullptr;
        ctx->stage_cap = 0;
        CK(cudaMalloc(&ctx->d_x, need * 8));
        CK(cudaMalloc(&ctx->d_y, need * 8));
        ctx->stage_cap = need;
      }
      CK(cudaMemcpy2DAsync(ctx->d_x, size_t(M) * 8, X, size_t(ldx) * 8, size_t(M) * 8, size_t(nrhs),
                           cudaMemcpyHostToDevice, st));
      hbs_apply(H, ctx->d_x, M, nrhs, ctx->d_y, M, st);
      CK(cudaMemcpy2DAsync(Y, size_t(ldy) * 8, ctx->d_y, size_t(M) * 8, size_t(M) * 8, size_t(nrhs),
                           cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

int dtn_gpu_hbs_serialize(const dtn_hbs* h, uint8_t* buf, uint64_t cap, uint64_t* size) {
  if (!h || !h->h || !size) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    CK(cudaSetDevice(ctx->device));
    *size = hbs_serialized_size(*h->h);  // a size query copies nothing
    if (!buf) return;
    if (cap < *size) throw std::invalid_argument("hbs_serialize: buffer too small");
    hbs_serialize_into(*h->h, buf, ctx->stream);
  });
}

int dtn_gpu_hbs_deserialize(dtn_ctx* ctx, const uint8_t* buf, uint64_t size, dtn_hbs** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (!buf) throw std::invalid_argument("deserialize: null buffer");
    CK(cudaSetDevice(ctx->device));
    auto hd = hbs_deserialize(buf, size_t(size), ctx->stream);
    auto* r = new dtn_hbs;
    r->ctx = ctx;
    r->h = std::move(hd);
    *out = r;
  });
}

int dtn_gpu_hbs_invert(const dtn_hbs* h, dtn_hbs** out) {
  if (!h || !h->h || !out) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(ctx->device));
    auto inv = hbs_invert(*h->h, ctx->stream);
    auto* r = new dtn_hbs;
    r->ctx = ctx;
    r->h = std::move(inv);
    *out = r;
  });
}

// ---- the HBS algebra (csrc/hbs_ops.cu): hbs.cpp:290-402, hbs_ops.cpp:213-743, lowrank.cpp
struct dtn_lowrank {
  dtn_ctx* ctx = nullptr;
  std::unique_ptr<LowRankDev> x;
};

namespace {

std::vector<HbsTreeNode> tree_from(const int64_t* nodes, int64_t num_nodes) {
  if (!nodes || num_nodes < 1 || num_nodes > (int64_t(1) << 24)) throw std::invalid_argument("index tree: no nodes");
  std::vector<HbsTreeNode> t(static_cast<size_t>(num_nodes));
  for (int64_t i = 0; i < num_nodes; ++i) {
    const int64_t* o = nodes + 6 * i;
    t[size_t(i)].begin = o[0];
    t[size_t(i)].end = o[1];
    t[size_t(i)].left = int(o[2]);
    t[size_t(i)].right = int(o[3]);
    t[size_t(i)].parent = int(o[4]);
    t[size_t(i)].level = int(o[5]);
  }
  return t;
}

// a host (or device) column-major matrix as a device pointer; host data staged into a
// pooled buffer the holder frees
struct DevMat {
  const double* p = nullptr;
  int64_t ld = 0;
  void* own = nullptr;
  DevMat(const double* src, int64_t lds, int64_t rows, int64_t cols, int on_device, cudaStream_t st) {
    if (rows > 0 && cols > 0 && (!src || lds < rows)) throw std::invalid_argument("matrix: null pointer or ld < rows");
    if (on_device || rows <= 0 || cols <= 0) {
      p = src;
      ld = std::max<int64_t>(lds, 1);
      return;
    }
    ld = (rows + 1) & ~int64_t(1);
    own = pool_alloc(size_t(ld) * size_t(cols) * 8);
    CK(cudaMemcpy2DAsync(own, size_t(ld) * 8, src, size_t(lds) * 8, size_t(rows) * 8, size_t(cols),
                         cudaMemcpyHostToDevice, st));
    p = static_cast<const double*>(own);
  }
  ~DevMat() { pool_free(own); }
};

dtn_hbs* wrap(dtn_ctx* ctx, std::unique_ptr<HbsDev> h) {
  auto* r = new dtn_hbs;
  r->ctx = ctx;
  r->h = std::move(h);
  return r;
}

dtn_lowrank* wrap_lr(dtn_ctx* ctx, std::unique_ptr<LowRankDev> x) {
  auto* r = new dtn_lowrank;
  r->ctx = ctx;
  r->x = std::move(x);
  return r;
}

}  // namespace

int dtn_gpu_hbs_compress_tree(dtn_ctx* ctx, const double* H, int64_t M, int64_t ldh, int on_device, double eps,
                              const int64_t* nodes, int64_t num_nodes, dtn_hbs** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (!H || M < 1 || ldh < M) throw std::invalid_argument("compress: matrix/tree size mismatch");
    CK(cudaSetDevice(ctx->device));
    const auto tree = tree_from(nodes, num_nodes);
    DevMat X(H, ldh, M, M, on_device, ctx->stream);
    *out = wrap(ctx, hbs_compress_tree(X.p, X.ld, M, eps, tree, ctx->stream));
  });
}

int dtn_gpu_hbs_reconstruct(const dtn_hbs* h, double* out, int64_t ldo, int on_device) {
  if (!h || !h->h || !out) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    const int64_t M = h->h->M;
    if (ldo < M) throw std::invalid_argument("reconstruct: ld < M");
    CK(cudaSetDevice(ctx->device));
    if (on_device) {
      hbs_dense(*h->h, out, ldo, ctx->stream);
      return;
    }
    const int64_t L = (M + 1) & ~int64_t(1);
    void* tmp = pool_alloc(size_t(L) * size_t(M) * 8);
    try {
      hbs_dense(*h->h, static_cast<double*>(tmp), L, ctx->stream);
      CK(cudaMemcpy2DAsync(out, size_t(ldo) * 8, tmp, size_t(L) * 8, size_t(M) * 8, size_t(M), cudaMemcpyDeviceToHost,
                           ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      pool_free(tmp);
      throw;
    }
    pool_free(tmp);
  });
}

int dtn_gpu_hbs_subtree(const dtn_hbs* h, int32_t node, dtn_hbs** out) {
  if (!h || !h->h || !out) return DTN_EINVAL;
  return guarded(h->ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(h->ctx->device));
    *out = wrap(h->ctx, hbs_subtree(*h->h, node, h->ctx->stream));
  });
}

int dtn_gpu_hbs_flip(const dtn_hbs* h, dtn_hbs** out) {
  if (!h || !h->h || !out) return DTN_EINVAL;
  return guarded(h->ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(h->ctx->device));
    *out = wrap(h->ctx, hbs_flip(*h->h, h->ctx->stream));
  });
}

namespace {
int scale_common(dtn_hbs* h, double s, const double* w, int on_device, int side) {
  if (!h || !h->h) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    CK(cudaSetDevice(ctx->device));
    const int64_t M = h->h->M;
    if (side != 0 && !w) throw std::invalid_argument("scale: null weights");
    DevMat W(w, M, M, side != 0 ? 1 : 0, on_device, ctx->stream);
    hbs_scale(*h->h, s, side == 1 ? W.p : nullptr, side == 2 ? W.p : nullptr, ctx->stream);
  });
}
}  // namespace

int dtn_gpu_hbs_scale(dtn_hbs* h, double s) { return scale_common(h, s, nullptr, 1, 0); }
int dtn_gpu_hbs_scale_rows(dtn_hbs* h, const double* w, int on_device) { return scale_common(h, 1.0, w, on_device, 1); }
int dtn_gpu_hbs_scale_cols(dtn_hbs* h, const double* w, int on_device) { return scale_common(h, 1.0, w, on_device, 2); }

int dtn_gpu_hbs_add(const dtn_hbs* A, const dtn_hbs* B, double eps, dtn_hbs** out) {
  if (!A || !A->h || !B || !B->h || !out) return DTN_EINVAL;
  return guarded(A->ctx, [&] {
    *out = nullptr;
    if (!(eps >= 0.0)) throw std::invalid_argument("add_hbs: eps must be >= 0");
    CK(cudaSetDevice(A->ctx->device));
    *out = wrap(A->ctx, hbs_add(*A->h, *B->h, eps, A->ctx->stream));
  });
}

int dtn_gpu_hbs_from_lowrank(dtn_ctx* ctx, const double* Q, int64_t ldq, const double* R, int64_t ldr, int64_t k,
                             const int64_t* nodes, int64_t num_nodes, int on_device, dtn_hbs** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(ctx->device));
    const auto tree = tree_from(nodes, num_nodes);
    const int64_t M = tree[0].end;
    if (k < 0) throw std::invalid_argument("lowrank_to_bs: negative rank");
    DevMat q(Q, ldq, M, k, on_device, ctx->stream), r(R, ldr, k, M, on_device, ctx->stream);
    *out = wrap(ctx, hbs_from_lowrank(q.p, q.ld, r.p, r.ld, k, tree, ctx->stream));
  });
}

int dtn_gpu_hbs_add_lowrank(const dtn_hbs* A, const double* Q, int64_t ldq, const double* R, int64_t ldr, int64_t k,
                            double eps, int on_device, dtn_hbs** out) {
  if (!A || !A->h || !out) return DTN_EINVAL;
  dtn_ctx* ctx = A->ctx;
  return guarded(ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(ctx->device));
    const int64_t M = A->h->M;
    if (k < 0) throw std::invalid_argument("add_lowrank: negative rank");
    DevMat q(Q, ldq, M, k, on_device, ctx->stream), r(R, ldr, k, M, on_device, ctx->stream);
    *out = wrap(ctx, hbs_add_lowrank(*A->h, q.p, q.ld, r.p, r.ld, k, eps, ctx->stream));
  });
}

int dtn_gpu_hbs_rebase(const dtn_hbs* h, const int64_t* nodes, int64_t num_nodes, double eps, dtn_hbs** out) {
  if (!h || !h->h || !out) return DTN_EINVAL;
  return guarded(h->ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(h->ctx->device));
    *out = wrap(h->ctx, hbs_rebase(*h->h, tree_from(nodes, num_nodes), eps, h->ctx->stream));
  });
}

int dtn_gpu_hbs_split_at(const dtn_hbs* h, int64_t pos, double eps, dtn_hbs** lo, dtn_hbs** hi, dtn_lowrank** lo_hi,
                         dtn_lowrank** hi_lo) {
  if (!h || !h->h || !lo || !hi || !lo_hi || !hi_lo) return DTN_EINVAL;
  dtn_ctx* ctx = h->ctx;
  return guarded(ctx, [&] {
    *lo = *hi = nullptr;
    *lo_hi = *hi_lo = nullptr;
    CK(cudaSetDevice(ctx->device));
    SplitDev sp = hbs_split_at(*h->h, pos, eps, ctx->stream);
    if (sp.lo) *lo = wrap(ctx, std::move(sp.lo));
    if (sp.hi) *hi = wrap(ctx, std::move(sp.hi));
    *lo_hi = wrap_lr(ctx, std::move(sp.lo_hi));
    *hi_lo = wrap_lr(ctx, std::move(sp.hi_lo));
  });
}

int dtn_gpu_hbs_consolidate(dtn_ctx* ctx, int64_t size, int64_t npieces, const dtn_hbs* const* pieces,
                            const int64_t* offsets, int64_t ncorr, const dtn_lowrank* const* corr,
                            const int64_t* corr_offsets, double eps, dtn_hbs** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (npieces < 1 || !pieces || !offsets) throw std::invalid_argument("consolidate: no pieces");
    if (ncorr < 0 || (ncorr > 0 && (!corr || !corr_offsets))) throw std::invalid_argument("consolidate: bad corrections");
    CK(cudaSetDevice(ctx->device));
    std::vector<const HbsDev*> p;
    std::vector<int64_t> o(offsets, offsets + npieces);
    for (int64_t i = 0; i < npieces; ++i) p.push_back(pieces[i] && pieces[i]->h ? pieces[i]->h.get() : nullptr);
    std::vector<LowRankPlaced> cs;
    for (int64_t i = 0; i < ncorr; ++i) {
      if (!corr[i] || !corr[i]->x) throw std::invalid_argument("consolidate: null correction");
      cs.push_back(LowRankPlaced{corr_offsets[2 * i], corr_offsets[2 * i + 1], corr[i]->x.get()});
    }
    *out = wrap(ctx, hbs_consolidate(size, p, o, cs, eps, ctx->stream));
  });
}

int dtn_gpu_lowrank_create(dtn_ctx* ctx, const double* Lf, int64_t ldl, const double* R, int64_t ldr, int64_t m,
                           int64_t n, int64_t k, int on_device, dtn_lowrank** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (m < 0 || n < 0 || k < 0) throw std::invalid_argument("lowrank: negative dimension");
    CK(cudaSetDevice(ctx->device));
    DevMat l(Lf, ldl, m, k, on_device, ctx->stream), r(R, ldr, k, n, on_device, ctx->stream);
    *out = wrap_lr(ctx, lowrank_from_factors(l.p, l.ld, r.p, r.ld, m, n, k, ctx->stream));
  });
}

int dtn_gpu_lowrank_from_dense(dtn_ctx* ctx, const double* X, int64_t ldx, int64_t m, int64_t n, int on_device,
                               double eps, dtn_lowrank** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (m < 0 || n < 0) throw std::invalid_argument("lowrank: negative dimension");
    CK(cudaSetDevice(ctx->device));
    DevMat x(X, ldx, m, n, on_device, ctx->stream);
    *out = wrap_lr(ctx, lowrank_from_dense(x.p, x.ld, m, n, eps, ctx->stream));
  });
}

int dtn_gpu_lowrank_info(const dtn_lowrank* x, int64_t* m, int64_t* n, int64_t* k) {
  if (!x || !x->x) return DTN_EINVAL;
  if (m) *m = x->x->m;
  if (n) *n = x->x->n;
  if (k) *k = x->x->k;
  return DTN_OK;
}

int dtn_gpu_lowrank_get(const dtn_lowrank* x, double* Lf, int64_t ldl, double* R, int64_t ldr) {
  if (!x || !x->x) return DTN_EINVAL;
  dtn_ctx* ctx = x->ctx;
  return guarded(ctx, [&] {
    const LowRankDev& a = *x->x;
    CK(cudaSetDevice(ctx->device));
    if (Lf && a.m > 0 && a.k > 0) {
      if (ldl < a.m) throw std::invalid_argument("lowrank_get: ldl < m");
      CK(cudaMemcpy2D(Lf, size_t(ldl) * 8, a.L, size_t(a.ldl) * 8, size_t(a.m) * 8, size_t(a.k), cudaMemcpyDeviceToHost));
    }
    if (R && a.k > 0 && a.n > 0) {
      if (ldr < a.k) throw std::invalid_argument("lowrank_get: ldr < k");
      CK(cudaMemcpy2D(R, size_t(ldr) * 8, a.R, size_t(a.ldr) * 8, size_t(a.k) * 8, size_t(a.n), cudaMemcpyDeviceToHost));
    }
  });
}

int dtn_gpu_lowrank_recompress(const dtn_lowrank* x, double eps, dtn_lowrank** out) {
  if (!x || !x->x || !out) return DTN_EINVAL;
  return guarded(x->ctx, [&] {
    *out = nullptr;
    CK(cudaSetDevice(x->ctx->device));
    *out = wrap_lr(x->ctx, lowrank_recompress(*x->x, eps, x->ctx->stream));
  });
}

int dtn_gpu_lowrank_sum(dtn_ctx* ctx, int64_t m, int64_t n, int64_t nterms, const dtn_lowrank* const* terms,
                        const int64_t* offsets, double eps, dtn_lowrank** out) {
  if (!ctx || !out) return DTN_EINVAL;
  return guarded(ctx, [&] {
    *out = nullptr;
    if (m < 0 || n < 0 || nterms < 0 || (nterms > 0 && (!terms || !offsets)))
      throw std::invalid_argument("lowrank_sum: bad arguments");
    CK(cudaSetDevice(ctx->device));
    std::vector<LowRankPlaced> t;
    for (int64_t i = 0; i < nterms; ++i) {
      if (!terms[i] || !terms[i]->x) throw std::invalid_argument("lowrank_sum: null term");
      t.push_back(LowRankPlaced{offsets[2 * i], offsets[2 * i + 1], terms[i]->x.get()});
    }
    *out = wrap_lr(ctx, lowrank_sum(m, n, t, eps, ctx->stream));
  });
}

void dtn_gpu_lowrank_free(dtn_lowrank* x) {
  if (!x) return;
  if (x->ctx) cudaSetDevice(x->ctx->device);
  delete x;
}

int dtn_gpu_build_accel(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, int64_t hbs_leaf, dtn_op** op_out,
                        dtn_hbs** S_hbs, dtn_hbs** G_hbs, double* cond) {
  if (!ctx || !prob || !opts || !S_hbs || !G_hbs) return DTN_EINVAL;
  *S_hbs = nullptr;
  *G_hbs = nullptr;
  if (op_out) *op_out = nullptr;
  if (!(opts->epsilon > 0.0) || hbs_leaf < 2) {
    ctx->err = "build_root_accel: epsilon must be > 0 and hbs_leaf >= 2";
    return DTN_EINVAL;
  }
  // the root is structured only when both of its W|E halves are: merge_pair
  // (accel_nd.cpp:667-689) compresses a merged box (size >= crossover) only when it
  // has a next merge (out_side != none), and the root's W|E merge has none
  // (accel_nd.cpp:771-779); a single-leaf tree stays dense
  bool dense_root = true;
  {
    PlanKey hk;
    hk.n = prob->n;
    hk.n_leaf = opts->n_leaf;
    hk.leaf_side = opts->leaf_side;
    int depth = 0, nb_w = 0, nb_e = 0;
    const int rc0 = guarded(ctx, [&] { root_halves(hk, &depth, &nb_w, &nb_e); });
    if (rc0 != DTN_OK) return rc0;
    dense_root = depth == 0 || nb_w < opts->crossover || nb_e < opts->crossover;
  }
  dtn_opts o = *opts;
  // engine 1: structured merges above the crossover (accel_merge on the B200); engine 0:
  // exact dense merges with only the root compressed. Body loads ride the dense merges.
  o.engine = (opts->engine == 1 && opts->nloads == 0) ? 1 : 0;
  o.want_G = dense_root ? 1 : 0;
  o.export_S = nullptr;
  dtn_op* op = nullptr;
  const bool trace = std::getenv("DTN_HBS_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(ctx->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[accel] %-10s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  int rc = dtn_gpu_build(ctx, prob, &o, &op);
  if (rc != DTN_OK) return rc;
  lap("build");
  if (dense_root) {  // accel_nd.cpp:796-818: below the crossover the accel engine holds dense factors
    if (cond) *cond = op->cond;
    if (op_out) *op_out = op;
    else dtn_gpu_free(op);
    return DTN_OK;
  }
  dtn_hbs* Sh = nullptr;
  dtn_hbs* Gh = nullptr;
  rc = dtn_gpu_hbs_compress_op(op, 1, opts->epsilon, hbs_leaf, &Sh);
  lap("compress");
  if (rc == DTN_OK) rc = dtn_gpu_hbs_invert(Sh, &Gh);  // accel_nd.cpp:820-822
  lap("invert");
  if (rc == DTN_OK && cond) {
    // accel_nd.cpp:834-841: (|S 1|_1 / m) (|G 1|_1 / m) m
    rc = guarded(ctx, [&] {
      const int64_t m = op->nb;
      std::vector<double> ones(size_t(m), 1.0);
      std::vector<double> y(2 * static_cast<size_t>(m), 0.0);
      double* d = static_cast<double*>(pool_alloc(size_t(m) * 24));
      struct F {
        double* p;
        ~F() { pool_free(p); }
      } f{d};
      cudaStream_t st = ctx->stream;
      CK(cudaMemcpyAsync(d, ones.data(), size_t(m) * 8, cudaMemcpyHostToDevice, st));
      // both products enqueued back to back, one copy back, one synchronisation
      hbs_apply(*Sh->h, d, m, 1, d + m, m, st, false);
      hbs_apply(*Gh->h, d, m, 1, d + 2 * m, m, st, false);
      CK(cudaMemcpyAsync(y.data(), d + m, size_t(m) * 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double nrm[2];
      for (int w = 0; w < 2; ++w) {
        double a = 0.0;
        for (int64_t i = 0; i < m; ++i) a += std::fabs(y[size_t(w * m + i)]);
        nrm[w] = a / double(m);
      }
      *cond = nrm[0] * nrm[1] * double(m);
    });
    lap("cond");
  }
  if (rc != DTN_OK) {
    dtn_gpu_hbs_free(Gh);
    dtn_gpu_hbs_free(Sh);
    dtn_gpu_free(op);
    return rc;
  }
  *S_hbs = Sh;
  *G_hbs = Gh;
  if (op_out) *op_out = op;
  else dtn_gpu_free(op);
  return DTN_OK;
}

}  // extern "C"
