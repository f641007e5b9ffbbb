// HBS (hierarchically block separable) matrices on the device: compression of
// a dense device-resident matrix, the telescoping apply, and the DTNHBS01
// byte format -- the reference's HbsMatrix (proj/include/dtn/hbs.hpp:30-51,
// proj/src/hbs.cpp) restated B200-first (see hbs.cu for the algorithm).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace dtnb {

struct TransDesc {  // dst (n x m) = src (m x n)^T
  const double* src;
  double* dst;
  int lds, ldd, m, n;
};

struct EigDesc {  // A (s x s, symmetric) -> diag(lambda) on its diagonal; V eigenvectors
  double* A;
  double* V;
  int s, lda, ldv;
};

struct SelDesc {  // lambda_i = lam[i * stride]; outputs order[s], sigma[s] (sorted), rank
  const double* lam;
  int* order;
  double* sigma;
  int* rank;
  int s, stride;
};

struct GatherDesc {  // dst(:, j) = src(:, order[j]), j < k
  const double* src;
  double* dst;
  const int* order;
  int lds, ldd, rows, k;
};

struct PackDesc {  // see pack_kernel (k_hbs.cu)
  const double* src;
  double* dst;
  int lds, ldd, rp, cp;
  int r1, rp1, r2, c1, cp1, c2;
  int trans;
};

struct ZeroDesc {
  double* p;
  int ld, m, n;
};

struct AddDesc {  // dst(m x n) += src(m x n)
  const double* src;
  double* dst;
  int lds, ldd, m, n;
};

struct InvDesc {  // A (s x s, leading dimension lda) <- A^{-1}; *info = 0, or k + 1 (singular at step k)
  double* A;
  int* info;
  int s, lda;
};

cudaError_t launch_transpose_batched(const TransDesc* d_descs, int count, int max_tiles, cudaStream_t st);
cudaError_t launch_jacobi_eig(const EigDesc* d_descs, int count, int max_sweeps, bool rel, double floor_rel,
                              int max_s, cudaStream_t st);
cudaError_t launch_hbs_select(const SelDesc* d_descs, int count, double eps, cudaStream_t st);
cudaError_t launch_gather_cols(const GatherDesc* d_descs, int count, cudaStream_t st);
cudaError_t launch_pack(const PackDesc* d_descs, int count, cudaStream_t st);
cudaError_t launch_zero_blocks(const ZeroDesc* d_descs, int count, cudaStream_t st);
cudaError_t launch_add_blocks(const AddDesc* d_descs, int count, cudaStream_t st);
cudaError_t launch_gj_inverse(const InvDesc* d_descs, int count, int max_s, cudaStream_t st);

// IndexTree node (index_tree.hpp:12-22): contiguous range [begin, end),
// preorder ids, children -1 for leaves.
// per-device caching device allocator of the compressed engine (hbs.cu)
void* pool_alloc(size_t bytes);
void pool_free(void* p);

struct HbsTreeNode {
  int64_t begin = 0, end = 0;
  int left = -1, right = -1, parent = -1, level = 0;
};

// build_index_tree (index_tree.cpp:37-67): balanced halving, the left half
// taking the extra index, ranges above leaf_cap split.
std::vector<HbsTreeNode> hbs_index_tree(int64_t M, int64_t leaf_cap, int* depth);

struct HbsDev {
  int device = 0;
  int64_t M = 0;
  int depth = 0;
  std::vector<HbsTreeNode> nodes;
  std::vector<int> rank;    // k_t (U/V columns); 0 for the root
  std::vector<int> rows;    // node_rows: leaf size, or k_left + k_right
  std::vector<int> height;  // 0 for leaves, 1 + max(children)
  // canonical factors (column-major, leading dimension ld(t) = rows rounded up
  // to even: every column 16-byte aligned for the DMMA GEMM), device
  std::vector<double*> D, U, V, B;
  int ld(int t) const { return int((rows[t] + 1) & ~1); }
  std::vector<void*> buffers;  // owning allocations
  // apply layout: ranks padded to even with zero columns, every block 16-byte aligned
  // apply layout (hbs.cu, pack_for_apply): per node a column group of the
  // transposed workspace -- leaf [x_t | y-hat_t], parent [x-hat_l x-hat_r | y-hat_t]
  struct Packed {
    bool ready = false;
    std::vector<int> kp, inner, go, gw, pb;  // padded rank, inner size, group offset/width, output offset
    int64_t cols = 0, out_cols = 0;
    std::vector<double*> V, W;  // V (inner x kp); W = [D^T; U^T] (leaf) or [B^T; U^T] (parent)
    std::vector<int> ldV, ldW;
    void* buf = nullptr;
  } pk;
  // apply workspace
  double* ws = nullptr;
  size_t ws_doubles = 0;
  int64_t ws_ld = 0;
  void* d_desc = nullptr;
  size_t desc_bytes = 0;
  // the apply's launch sequence as a CUDA graph (valid for one batch size and
  // descriptor buffer; the descriptors themselves are re-uploaded every call)
  cudaGraphExec_t apply_graph = nullptr;
  int64_t apply_graph_nrhs = -1;
  const void* apply_graph_desc = nullptr;
  ~HbsDev();
  int64_t max_rank() const;
  uint64_t payload_bytes() const;
  bool is_leaf(int t) const { return nodes[t].left < 0; }
  int64_t node_size(int t) const { return nodes[t].end - nodes[t].begin; }
};

// compress (hbs.cpp:61-178): dense H (M x M, column-major, leading dimension
// ldh, device memory) onto build_index_tree(M, leaf_cap) with relative
// tolerance eps. Throws std::invalid_argument / std::runtime_error.
std::unique_ptr<HbsDev> hbs_compress(const double* dH, int64_t ldh, int64_t M, double eps, int64_t leaf_cap,
                                     cudaStream_t st);

// compress(H, tree, eps) (hbs.hpp:58-60, hbs.cpp:61-178) onto a given index tree
// (preorder, children partition their parent: checked, std::invalid_argument).
std::unique_ptr<HbsDev> hbs_compress_tree(const double* dH, int64_t ldh, int64_t M, double eps,
                                          const std::vector<HbsTreeNode>& tree, cudaStream_t st);
void hbs_check_tree(const std::vector<HbsTreeNode>& nodes, int64_t M, const char* what);

// Y (M x nrhs) = H X through the telescoping factorization (hbs.cpp:187-232);
// X, Y device pointers.
// allow_graph = false: launch the sweep directly (one-off applies: capturing and
// instantiating the per-batch-size graph costs more than it saves)
void hbs_apply(HbsDev& H, const double* dX, int64_t ldx, int64_t nrhs, double* dY, int64_t ldy, cudaStream_t st,
               bool allow_graph = true);

// A singular block met by hbs_invert: what() = "<what> [node t level l]"
// (FactorizationError, errors.hpp:11-21); the C ABI maps it to DTN_ESINGULAR.
struct HbsSingular : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// invert_hbs (hbs_ops.cpp:148-201): the telescoping inverse factors of H on
// the same tree -- E in U, F in V, G in D (leaves) / B (parents), the root
// core inverse (B_root + diag(Dhat))^{-1} in the root B -- so hbs_apply on
// the result is apply_inverse (hbs_ops.cpp:203-205).
std::unique_ptr<HbsDev> hbs_invert(const HbsDev& H, cudaStream_t st);

// ---- the HBS algebra (hbs_ops.cu): hbs.cpp:290-402, hbs_ops.cpp:213-743, lowrank.cpp
// Low-rank block L R (L m x k, R k x n, column-major, device; LowRank, lowrank.hpp).
struct LowRankDev {
  int device = -1;
  int64_t m = 0, n = 0, k = 0, ldl = 2, ldr = 2;
  double* L = nullptr;
  double* R = nullptr;
  void* buf = nullptr;
  LowRankDev() = default;
  LowRankDev(const LowRankDev&) = delete;
  LowRankDev& operator=(const LowRankDev&) = delete;
  ~LowRankDev();
};
struct LowRankPlaced {  // PlacedLowRank (lowrank.hpp): a block at (row_offset, col_offset)
  int64_t row_offset = 0, col_offset = 0;
  const LowRankDev* lr = nullptr;
};
struct SplitDev {  // SplitParts (hbs_ops.hpp) with both accumulations consolidated
  std::unique_ptr<HbsDev> lo, hi;
  std::unique_ptr<LowRankDev> lo_hi, hi_lo;
};
std::unique_ptr<HbsDev> hbs_subtree(const HbsDev& H, int t, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_copy(const HbsDev& H, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_flip(const HbsDev& H, cudaStream_t st);
void hbs_scale(HbsDev& H, double s, const double* d_wrow, const double* d_wcol, cudaStream_t st);
void hbs_dense(const HbsDev& H, double* dX, int64_t ldx, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_add(const HbsDev& A, const HbsDev& B, double eps, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_from_lowrank(const double* dQ, int64_t ldq, const double* dR, int64_t ldr, int64_t k,
                                         const std::vector<HbsTreeNode>& tree, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_add_lowrank(const HbsDev& A, const double* dQ, int64_t ldq, const double* dR, int64_t ldr,
                                        int64_t k, double eps, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_rebase(const HbsDev& H, const std::vector<HbsTreeNode>& target, double eps,
                                   cudaStream_t st);
SplitDev hbs_split_at(const HbsDev& H, int64_t pos, double eps, cudaStream_t st);
std::unique_ptr<HbsDev> hbs_consolidate(int64_t size, const std::vector<const HbsDev*>& pieces,
                                        const std::vector<int64_t>& offsets, const std::vector<LowRankPlaced>& corr,
                                        double eps, cudaStream_t st);
std::unique_ptr<LowRankDev> lowrank_alloc(int64_t m, int64_t n, int64_t k);
std::unique_ptr<LowRankDev> lowrank_from_factors(const double* dL, int64_t ldl, const double* dR, int64_t ldr,
                                                 int64_t m, int64_t n, int64_t k, cudaStream_t st);
std::unique_ptr<LowRankDev> lowrank_recompress(const LowRankDev& x, double eps, cudaStream_t st);
std::unique_ptr<LowRankDev> lowrank_from_dense(const double* dX, int64_t ldx, int64_t m, int64_t n, double eps,
                                               cudaStream_t st);
std::unique_ptr<LowRankDev> lowrank_sum(int64_t m, int64_t n, const std::vector<LowRankPlaced>& terms, double eps,
                                        cudaStream_t st);

// DTNHBS01 serialization (hbs.cpp:422-519), byte-for-byte the reference layout.
std::vector<uint8_t> hbs_serialize(const HbsDev& H, cudaStream_t st);
uint64_t hbs_serialized_size(const HbsDev& H);
void hbs_serialize_into(const HbsDev& H, uint8_t* buf, cudaStream_t st);  // buf: hbs_serialized_size bytes
std::unique_ptr<HbsDev> hbs_deserialize(const uint8_t* data, size_t size, cudaStream_t st);

}  // namespace dtnb
