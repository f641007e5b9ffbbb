// Build plan for the B200 dense engine: the quadtree of the reference
// (proj/src/grid.cpp:213-266, or an exact-halving uniform variant), extended
// below its leaves by binary splits down to "micro boxes" small enough to be
// eliminated by one CTA, turned into a DAG of pairwise merges scheduled in
// waves (all merges of a wave are independent and run as one batched launch).
//
// Everything here is coefficient-independent (it depends only on n and the
// tree parameters), so a plan is built once and cached per context.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dtnb {

struct Rect {
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;  // inclusive unknown rectangle
  int w() const { return x1 - x0 + 1; }
  int h() const { return y1 - y0 + 1; }
  bool empty() const { return x0 > x1 || y0 > y1; }
  int64_t nodes() const { return empty() ? 0 : int64_t(w()) * h(); }
};

// CCW perimeter from the SW corner (grid.cpp:170-190); degenerate 1-wide
// rectangles are a single scan.
void perimeter_ccw(const Rect& r, std::vector<std::pair<int, int>>& out);
int perimeter_size(const Rect& r);

// Reference quadtree box (grid.hpp:120-141); children SW, SE, NW, NE.
struct RefBox {
  int id = -1, level = 0, parent = -1;
  int children[4] = {-1, -1, -1, -1};
  int gx0 = 0, gx1 = 0, gy0 = 0, gy1 = 0;
  Rect r;
  int node = -1;  // DAG node holding this box's Schur complement
};

// A device-side position descriptor of a merge or micro box: one per row of
// the assembled system, in the order [interior; boundary(CCW)].
struct PosEntry {
  int32_t src;      // merge: >=0 index in child a's boundary, <0: -(index in b)-1
                    // micro: unused (0)
  int32_t partner;  // merge: position of the node coupled across the interface, or -1
  int32_t gid;      // unknown id of this node
  int32_t dir;      // merge: stencil direction of the coupling (1=E,2=W,3=N,4=S), 0 if none
};

enum class NodeKind : int { micro = 0, merge = 1 };

struct Node {
  NodeKind kind = NodeKind::micro;
  Rect r;
  int nb = 0;        // boundary size = perimeter_size(r)
  int ni = 0;        // eliminated unknowns (micro: interior; merge: interface)
  int total = 0;     // ni + nb (rows of the assembled system)
  int a = -1, b = -1;  // children (merge)
  int wave = 0;
  int ref_box = -1;    // reference box id when this node is one
  int label_level = -1, label_box = -1;  // error label (dense_nd.cpp:16-18)
  bool blocked = false;  // assembled in HBM and eliminated by the blocked kernels
  // storage (offsets in doubles into the plan arena)
  int64_t s_off = 0;   // S block (nb x nb, leading dimension ld)
  int ld = 0;
  int64_t m_off = 0;   // blocked: assembled system (total x total, leading dim ldm)
  int ldm = 0;
  int64_t pos_off = 0;  // offset into the PosEntry table
  int64_t piv_off = 0;  // blocked: offset into the int pivot table
  int64_t uinv_off = 0;  // blocked: inverses of the 128 x 128 diagonal blocks of U (back substitution)
  int64_t t_off = 0;     // blocked: 128 x nb staging block of the back substitution
  // body-load right-hand sides (dense_nd.hpp:18-26 `rhs`, nb x nloads): compact
  // for micro/small nodes, the view M[ni:total, total:total+nloads] for blocked ones
  int64_t rhs_off = 0;
  int rhs_ld = 0;
  // ---- compressed engine (build_root_accel, accel_nd.cpp:667-689, 707-859) ----
  // A structured box keeps its S dense in CCW order plus rank-ell factors of the
  // off-diagonal blocks of its [J; K] split (StructuredSchur, accel_nd.hpp:31-48;
  // J = the edge eliminated at the box's next merge, arc_boundary :46-88):
  //   S[J, K] ~= Q1 (Q1^T S[J, :])  -> L_jk = Q1 (jn x ell), R_jk^T = S[J, :]^T Q1 (nb x ell)
  //   S[K, J] ~= (S[:, J] Q2) Q2^T  -> L_kj = S[:, J] Q2 (nb x ell), R_kj^T = Q2 (jn x ell)
  // A structured merge (accel_merge :434-628) factors only the reduced interface
  // system [[M_jj, Z], [W, 0]] (Z = blockdiag(L_jk), W = blockdiag(R_kj)) and adds
  // the rank-(ra + rb) product L_k C R_k to the assembled kept block.
  int parent = -1;       // consumer merge node (-1: the root / a shard root)
  int jside = -1;        // 0 north, 1 south, 2 east, 3 west; -1: no next merge (root)
  bool factors = false;  // structured box: factors formed at the end of its wave
  bool smerge = false;   // structured merge (both children structured)
  bool exact = false;    // structured box whose factors would be full rank: kept dense (exact)
  bool colshard = false; // collective top build: boundary columns split over the ranks
  int cw = 0;            // column chunk per rank (ceil(nb / world))
  int j0 = 0, jn = 0;    // J edge = positions [j0, j0 + jn) of the CCW boundary
  int ell = 0;           // factor rank (randomized range-finder sketch width)
  int sys_nb = 0;        // boundary columns of the blocked system: nb, or ra + rb (smerge)
  int pos_n = 0;         // rows of the position table (ni + nb)
  int64_t q1_off = 0, q2_off = 0, rt_off = 0, lk_off = 0;
  int ldq = 0, ldf = 0;
  // scratch of the node's own wave: sketch (omega nb x ell, y1 / y2 jn x ell);
  // structured merge: gathered L_k, R_k^T and T = L_k C (nb x (ra + rb) each)
  int64_t om_off = 0, y1_off = 0, y2_off = 0, lkg_off = 0, rkg_off = 0, tg_off = 0, cbuf_off = 0;
  int ldg = 0, ldr = 0;
  // the sketches Y1 / Y2 (K = nb) split into ysplit K-slices: slice 0 into y1 / y2, the
  // others into partials (ysp_off: per slice [Y1 part | Y2 part], ldq x (ell + 4) each)
  int ysplit = 1;
  int64_t ysp_off = 0;
};

struct Wave {
  std::vector<int> micro, small, blocked;  // node ids (blocked: dense blocked merges and structured merges)
  std::vector<int> smerge;                 // the structured merges among `blocked`
  std::vector<int> compress;               // structured boxes whose factors are formed at the end of the wave
  int max_ni_blocked = 0;
};

// Subtree sharding: nshards in {1, 2, 4, 8} splits the tree into
// the root's W|E halves, its quadrants, or the quadrants' W|E halves.
// shard >= 0: build only that shard's subtree (its S is the result);
// shard == -1 with nshards > 1: the top of the tree above the shards, whose
// S blocks are inputs.
struct PlanKey {
  int n = 0, n_leaf = 0, leaf_side = 0, micro_max = 0, small_max = 0;
  int nshards = 1, shard = -1;
  int nloads = 0;  // body-load columns carried through the merges (LoadPanel, dense_nd.hpp:29-32)
  // compressed engine: boxes of boundary >= crossover with a next merge become
  // structured (accel_nd.cpp:682, 737); factor rank ell(jn) = min(jn, ell_base +
  // ell_step * floor(log2(jn / 128))) rounded up to a multiple of 8
  int structured = 0;
  int64_t crossover = 0;
  int ell_base = 0, ell_step = 0;
  int keep = 0;  // keep every box's S resident (dtn_gpu_box_schur); else storage is reused level by level
  // learned ranks: (J edge size, ell) overrides of the schedule, raised by the engine when a
  // factor's range-finder check fails (engine.cu, dtn_gpu_build)
  std::vector<std::pair<int, int>> ell_over;
  // collective top build: the blocked merges above the shards are
  // column-sharded over `world` ranks -- interface LU redundant on every rank, the
  // boundary columns' substitutions and Schur GEMM split in `world` chunks of
  // ceil(nb / world) columns, gathered after each wave (ncclAllGather). wrank: this
  // rank's chunk, or -1: every chunk computed locally (single-device check of the split)
  int world = 1, wrank = -1;
  bool operator==(const PlanKey& o) const {
    return n == o.n && n_leaf == o.n_leaf && leaf_side == o.leaf_side && micro_max == o.micro_max &&
           small_max == o.small_max && nshards == o.nshards && shard == o.shard && nloads == o.nloads &&
           structured == o.structured && crossover == o.crossover && ell_base == o.ell_base &&
           ell_step == o.ell_step && keep == o.keep && ell_over == o.ell_over && world == o.world &&
           wrank == o.wrank;
  }
};

struct Plan {
  PlanKey key;
  int n = 0;
  int depth = 0;
  std::vector<RefBox> boxes;
  std::vector<std::vector<int>> levels;
  std::vector<Node> nodes;
  std::vector<Wave> waves;
  std::vector<PosEntry> pos;  // all position tables
  int64_t arena_doubles = 0;
  int64_t piv_ints = 0;
  int root = -1;  // root node (the shard's node in shard mode)
  std::vector<int> inputs;  // top mode: shard nodes whose S is provided by the caller
  std::vector<char> active;  // nodes computed by this plan
  int64_t arena_peak_bytes = 0;  // liveness-packed arena (vs the sum of all node storage)
  int64_t arena_sum_bytes = 0;
  // algorithmic work (reference formulation)
  double merge_flops = 0.0;     // sum of (2/3)ni^3 + 2ni^2nb + 2nb^2ni over reference-tree merges
  double micro_flops = 0.0;     // leaf-interior elimination executed (same formula)
};

// Builds the plan; leaf_side > 0 selects the uniform tree (n-2 = leaf_side*2^L),
// else the reference rule with n_leaf. Throws std::invalid_argument.
Plan make_plan(const PlanKey& key);

// Depth of the reference tree and the boundary sizes of the root's W and E
// halves (merge_four's (SW,NW) and (SE,NE) merges, dense_nd.cpp:188-194);
// host-only, no DAG. The compressed engine's root is structured only when both
// halves are (accel_nd.cpp:667-689, 771-779).
void root_halves(const PlanKey& key, int* depth, int* nb_w, int* nb_e);

// DAG nodes of the shards of a full plan (see PlanKey), in shard order.
std::vector<int> shard_nodes(const Plan& P, int nshards);

inline double merge_flop_count(double ni, double nb) {
  return (2.0 / 3.0) * ni * ni * ni + 2.0 * ni * ni * nb + 2.0 * nb * nb * ni;
}

}  // namespace dtnb
