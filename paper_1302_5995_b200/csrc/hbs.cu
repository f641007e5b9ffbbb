// HBS compression and apply on the device (the reference's hbs.cpp:61-232 and
// its DTNHBS01 format, hbs.cpp:422-519), organised for the GPU.
//
// compress (hbs.cpp:61-178) keeps a "frontier" of already-compressed nodes
// covering [0, M) and the reduced matrix R(f, g) = Ubig_f^T H(I_f, I_g) Vbig_g
// (f != g), merging sibling pairs bottom up. Here the frontier is advanced one
// tree height at a time, every node of that height at once: with X the current
// reduced matrix (H itself for the leaves),
//   1. the active diagonal blocks are taken out (leaf D, parent B) and zeroed,
//   2. per active node f, the bases of the block row X(f, :) and the block
//      column X(:, f) are the leading left singular vectors of those blocks
//      (hbs.cpp:42-57 node_bases, shared rank = max of the two eps-ranks,
//      hbs.cpp:33-40). Singular values are needed to eps = 1e-10 relative, so
//      a plain Gram matrix (accurate to sqrt(machine eps)) is not enough: the
//      block is first rotated by the eigenvectors U0 of its Gram matrix
//      G1 = A A^T (Jacobi), which grades its rows by singular value
//      (B = U0^T A); the Gram matrix of B, G2 = B B^T, is then diagonalised by
//      Jacobi with the relative stopping rule, which resolves every singular
//      value to relative accuracy (U = U0 W). All products are DMMA GEMMs.
//   3. X' = blockdiag(U)^T X blockdiag(V) (identity blocks for nodes not yet
//      active) is the next reduced matrix; its active diagonal blocks are
//      exactly zero.
// The result is an orthonormal-basis HBS matrix of the reference's structure
// (D leaves, U/V non-root, B parents). Ranks and bases agree with the
// reference's BDCSVD-based compress up to rounding (same eps rule); the
// processing order (by height instead of reverse preorder) changes only
// which already-truncated columns a node's block row sees, i.e. results at
// the eps level.
//
// apply (hbs.cpp:187-232): upward x-hat = V^T x, root/parents B, downward
// U y-hat, leaves D x + U y-hat; batched DMMA GEMMs per tree height on a
// repacked copy of the factors whose ranks are padded to even (zero columns)
// so every operand is 16-byte aligned.
#include <atomic>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <stdexcept>

#include "common.cuh"
#include "hbs.hpp"

namespace dtnb {

// Device memory of the compressed engine comes from a per-device caching pool:
// cudaMalloc/cudaFree next to a large resident build (a 100+ GB plan arena)
// were measured to stall for tens of ms at random, and cudaFree synchronises
// the device. Freed blocks are kept (best fit, at most 2x the request + 1 MB)
// and returned to the driver only when an allocation fails.
namespace {
struct DevPool {
  std::mutex m;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> live_;
};
DevPool& dev_pool(int device) {
  static DevPool pools[64];
  return pools[device & 63];
}
}  // namespace

void* pool_alloc(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool& P = dev_pool(dev);
  bytes = (std::max<size_t>(bytes, 256) + 255) & ~size_t(255);
  {
    std::lock_guard<std::mutex> lk(P.m);
    auto it = P.free_.lower_bound(bytes);
    if (it != P.free_.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
      void* p = it->second;
      P.live_[p] = it->first;
      P.free_.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {  // give the cached blocks back and retry once
    (void)cudaGetLastError();
    std::lock_guard<std::mutex> lk(P.m);
    for (auto& kv : P.free_) cudaFree(kv.second);
    P.free_.clear();
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " (pool_alloc)");
  std::lock_guard<std::mutex> lk(P.m);
  P.live_[p] = bytes;
  return p;
}

void pool_free(void* p) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  DevPool& P = dev_pool(dev);
  std::lock_guard<std::mutex> lk(P.m);
  auto it = P.live_.find(p);
  if (it == P.live_.end()) {  // not from the pool
    cudaFree(p);
    return;
  }
  P.free_.insert({it->second, p});
  P.live_.erase(it);
}

}  // namespace dtnb

#include "hbs_impl.hpp"

namespace dtnb {

// kernel launches issued by the HBS code (compress, invert, apply, algebra), process-wide
std::atomic<unsigned long long> g_hbs_launches{0};

Scratch& scratch(int device) {
  static Scratch s[64];
  return s[device & 63];
}

namespace {

// DTN_HBS_TRACE=1: per-phase host timings of compress (after each synchronisation)
struct Trace {
  bool on = std::getenv("DTN_HBS_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> acc;
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t - t0).count();
    t0 = t;
    for (auto& a : acc)
      if (a.first == what) {
        a.second += ms;
        return;
      }
    acc.push_back({what, ms});
  }
  ~Trace() {
    if (!on) return;
    for (auto& a : acc) std::fprintf(stderr, "[hbs] %-12s %9.3f ms\n", a.first.c_str(), a.second);
  }
};

}  // namespace

// ---------------------------------------------------------------------------
std::vector<HbsTreeNode> hbs_index_tree(int64_t M, int64_t leaf_cap, int* depth) {
  if (M < 1) throw std::invalid_argument("build_index_tree: M must be >= 1");
  if (leaf_cap < 2) throw std::invalid_argument("build_index_tree: leaf_cap must be >= 2");
  std::vector<HbsTreeNode> nodes;
  int dmax = 0;
  // preorder: node, left subtree, right subtree (index_tree.cpp:39-52)
  struct Frame {
    int64_t b, e;
    int parent, level, side;
  };
  std::vector<Frame> stack{{0, M, -1, 0, 0}};
  while (!stack.empty()) {
    const Frame f = stack.back();
    stack.pop_back();
    const int id = int(nodes.size());
    HbsTreeNode n;
    n.begin = f.b;
    n.end = f.e;
    n.parent = f.parent;
    n.level = f.level;
    nodes.push_back(n);
    dmax = std::max(dmax, f.level);
    if (f.parent >= 0) (f.side == 0 ? nodes[f.parent].left : nodes[f.parent].right) = id;
    if (f.e - f.b > leaf_cap) {
      const int64_t mid = f.b + (f.e - f.b + 1) / 2;
      stack.push_back({mid, f.e, id, f.level + 1, 1});  // right popped after the whole left subtree
      stack.push_back({f.b, mid, id, f.level + 1, 0});
    }
  }
  if (depth) *depth = dmax;
  return nodes;
}

HbsDev::~HbsDev() {
  if (device >= 0) cudaSetDevice(device);
  for (void* p : buffers) pool_free(p);
  if (pk.buf) pool_free(pk.buf);
  if (ws) pool_free(ws);
  if (d_desc) pool_free(d_desc);
  if (apply_graph) cudaGraphExecDestroy(apply_graph);
}

int64_t HbsDev::max_rank() const {
  int64_t k = 0;
  for (size_t t = 1; t < nodes.size(); ++t) k = std::max<int64_t>(k, rank[t]);
  return k;
}

uint64_t HbsDev::payload_bytes() const {
  uint64_t n = 0;
  for (size_t t = 0; t < nodes.size(); ++t) {
    if (is_leaf(int(t))) n += uint64_t(node_size(int(t))) * uint64_t(node_size(int(t)));
    if (t != 0) n += 2 * uint64_t(rows[t]) * uint64_t(rank[t]);
    if (!is_leaf(int(t))) n += uint64_t(rows[t]) * uint64_t(rows[t]);
  }
  return n * sizeof(double);
}

// ---------------------------------------------------------------------------
// DTN_HBS_JACOBI=1: the round-1 bases (Gram + two-pass relative Jacobi eigensolves)
// instead of the randomized rank-revealing QR
bool use_jacobi_bases() {
  static const bool v = std::getenv("DTN_HBS_JACOBI") != nullptr;
  return v;
}

std::unique_ptr<HbsDev> hbs_compress(const double* dH, int64_t ldh, int64_t M, double eps, int64_t leaf_cap,
                                     cudaStream_t st) {
  if (M < 1 || ldh < M) throw std::invalid_argument("compress: matrix/tree size mismatch");
  int depth = 0;
  auto nodes = hbs_index_tree(M, leaf_cap, &depth);
  return hbs_compress_tree(dH, ldh, M, eps, nodes, st);
}

void hbs_check_tree(const std::vector<HbsTreeNode>& nodes, int64_t M, const char* what) {
  const std::string w = std::string(what) + ": ";
  const int64_t nn = int64_t(nodes.size());
  if (nn < 1 || nodes[0].begin != 0 || nodes[0].end != M || nodes[0].parent != -1)
    throw std::invalid_argument(w + "tree does not cover [0, M)");
  for (int t = 0; t < int(nn); ++t) {
    const auto& n = nodes[size_t(t)];
    if ((n.left < 0) != (n.right < 0) || n.left >= nn || n.right >= nn || n.left == 0 || n.right == 0)
      throw std::invalid_argument(w + "bad tree");
    if (n.begin < 0 || n.end <= n.begin || n.end > M) throw std::invalid_argument(w + "bad tree");
    if (n.left >= 0) {  // children partition the parent's range, preorder ids (index_tree.cpp:37-67)
      const auto& l = nodes[size_t(n.left)];
      const auto& r = nodes[size_t(n.right)];
      if (n.left <= t || n.right <= t || l.parent != t || r.parent != t || l.begin != n.begin || l.end != r.begin ||
          r.end != n.end || l.level != n.level + 1 || r.level != n.level + 1)
        throw std::invalid_argument(w + "bad tree");
    }
  }
}

std::unique_ptr<HbsDev> hbs_compress_tree(const double* dH, int64_t ldh, int64_t M, double eps,
                                          const std::vector<HbsTreeNode>& tree, cudaStream_t st) {
  if (M < 1 || ldh < M) throw std::invalid_argument("compress: matrix/tree size mismatch");
  if (!(eps >= 0.0)) throw std::invalid_argument("compress: eps must be >= 0");
  if (M > (int64_t(1) << 30) / 2) throw std::invalid_argument("compress: matrix too large");
  hbs_check_tree(tree, M, "compress");
  auto out = std::make_unique<HbsDev>();
  HbsDev& H = *out;
  HCK(cudaGetDevice(&H.device));
  H.M = M;
  H.nodes = tree;
  H.depth = 0;
  for (const auto& n : tree) H.depth = std::max(H.depth, n.level);
  int64_t leaf_cap = 2;  // scratch sizing: the largest leaf
  for (int t = 0; t < int(tree.size()); ++t)
    if (tree[size_t(t)].left < 0) leaf_cap = std::max<int64_t>(leaf_cap, tree[size_t(t)].end - tree[size_t(t)].begin);
  const int nn = int(H.nodes.size());
  H.rank.assign(nn, 0);
  H.rows.assign(nn, 0);
  H.height.assign(nn, 0);
  H.D.assign(nn, nullptr);
  H.U.assign(nn, nullptr);
  H.V.assign(nn, nullptr);
  H.B.assign(nn, nullptr);
  for (int t = nn - 1; t >= 0; --t)  // children have larger preorder ids
    if (!H.is_leaf(t)) H.height[t] = 1 + std::max(H.height[H.nodes[t].left], H.height[H.nodes[t].right]);
  DevBuf dbuf;
  if (nn == 1) {  // stored densely (hbs.cpp:75-78)
    H.rows[0] = int(M);
    double* d = nullptr;
    pmalloc(&d, size_t(H.ld(0)) * M * 8);
    H.buffers.push_back(d);
    H.D[0] = d;
    copy_batch(dbuf, {CopyDesc{dH, d, int(ldh), H.ld(0), int(M), int(M)}}, st);
    HCK(cudaStreamSynchronize(st));
    return out;
  }

  // work buffers (ld = align2(M) everywhere; every slot column block 16-byte aligned)
  const int64_t L = align2(M);
  const size_t big = size_t(L) * size_t(M);
  double *X = nullptr, *XT = nullptr, *P1 = nullptr, *P2 = nullptr, *Q1 = nullptr, *Q2 = nullptr;
  struct Frees {
    std::vector<void*> v;
    ~Frees() {
      for (void* p : v) pool_free(p);
    }
  } frees;
  Scratch& scr = scratch(H.device);
  std::lock_guard<std::mutex> lock(scr.m);
  Trace tr;
  // factors: leaf D (M x leaf) plus bases/couplings of ranks ~ leaf size; grown on demand
  Arena arena(H, size_t(align2(M)) * size_t(std::min<int64_t>(leaf_cap, M)) * 4);
  {
    int i = 0;
    for (double** p : {&X, &XT, &P1, &P2}) *p = static_cast<double*>(scr.get(i++, big * 8));
  }
  // B blocks (align2(s) x nX each, all active nodes): up to (M + nodes) x M
  const size_t qbig = size_t(M + nn) * size_t(M) + 64;
  Q1 = static_cast<double*>(scr.get(4, qbig * 8));
  Q2 = static_cast<double*>(scr.get(5, qbig * 8));
  tr.mark("alloc");
  // X = H
  copy_batch(dbuf, {CopyDesc{dH, X, int(ldh), int(L), int(M), int(M)}}, st);
  int64_t nX = M, ldX = L;

  // frontier: node ids in index order with their slot offsets and sizes
  std::vector<int> slots;
  for (int t = 0; t < nn; ++t)
    if (H.is_leaf(t)) slots.push_back(t);
  std::sort(slots.begin(), slots.end(), [&](int a, int b) { return H.nodes[a].begin < H.nodes[b].begin; });
  std::vector<int> ssize(nn, 0);
  for (int t : slots) ssize[t] = int(H.node_size(t));
  const int R = H.height[0];

  for (int r = 0; r <= R; ++r) {
    // parents of height r take their children's adjacent slots
    if (r > 0) {
      std::vector<int> ns;
      for (size_t i = 0; i < slots.size(); ++i) {
        const int t = slots[i], p = H.nodes[t].parent;
        if (p >= 0 && H.height[p] == r && H.nodes[p].left == t) {
          if (i + 1 >= slots.size() || slots[i + 1] != H.nodes[p].right)
            throw std::logic_error("compress: children not adjacent in frontier");
          ns.push_back(p);
          ssize[p] = ssize[t] + ssize[slots[i + 1]];
          H.rows[p] = ssize[p];
          ++i;
        } else {
          ns.push_back(t);
        }
      }
      slots.swap(ns);
    }
    std::vector<int64_t> off(slots.size());
    {
      int64_t o = 0;
      for (size_t i = 0; i < slots.size(); ++i) {
        off[i] = o;
        o += ssize[slots[i]];
      }
      if (o != nX) throw std::logic_error("compress: frontier size mismatch");
    }
    std::vector<int> act;  // frontier positions of this round's nodes
    for (size_t i = 0; i < slots.size(); ++i)
      if (H.height[slots[i]] == r) act.push_back(int(i));

    if (r == R) {  // the root: B = the reduced matrix of its two children (hbs.cpp:122-125)
      double* b = nullptr;
      H.rows[0] = int(nX);
      b = arena.alloc(size_t(H.ld(0)) * nX + 2);
      H.B[0] = b;
      copy_batch(dbuf, {CopyDesc{X, b, int(ldX), H.ld(0), int(nX), int(nX)}}, st);
      break;
    }

    // 1. diagonal blocks out (leaf D / parent B), then zeroed
    size_t diag_doubles = 0;
    for (int i : act) diag_doubles += size_t(align2(ssize[slots[i]])) * ssize[slots[i]];
    double* dbase = nullptr;
    dbase = arena.alloc(diag_doubles + 2);
    {
      std::vector<CopyDesc> cp;
      std::vector<ZeroDesc> zd;
      size_t o = 0;
      for (int i : act) {
        const int t = slots[i], s = ssize[t];
        double* dst = dbase + o;
        o += size_t(align2(s)) * s;
        (H.is_leaf(t) ? H.D[t] : H.B[t]) = dst;
        H.rows[t] = s;
        double* blk = X + off[i] + off[i] * ldX;
        cp.push_back(CopyDesc{blk, dst, int(ldX), int(align2(s)), s, s});
        zd.push_back(ZeroDesc{blk, int(ldX), s, s});
      }
      copy_batch(dbuf, cp, st);
      ZeroDesc* dz = upload(dbuf, zd, st);
      HLK(launch_zero_blocks(dz, int(zd.size()), st));
    }
    tr.mark("diag");
    // 2. XT = X^T
    transpose_batch(dbuf, {TransDesc{X, XT, int(ldX), int(ldX), int(nX), int(nX)}}, st);

    // per active node and side (0: rows -> U, 1: columns -> V): work layout
    const int na = int(act.size());
    std::vector<size_t> goff(na);
    size_t gsum = 0;
    int smax = 0;
    for (int a = 0; a < na; ++a) {
      const int s = ssize[slots[act[a]]];
      goff[a] = gsum;
      gsum += size_t(align2(s)) * s;
      smax = std::max(smax, s);
    }
    if (smax > 1024) throw std::runtime_error("compress: block of more than 1024 rows (rank too high)");
    // G1 (2 sides), U0, G2, W, Ufull: 2 * 5 * gsum doubles; select outputs
    double* wk = static_cast<double*>(scr.get(6, (10 * gsum + 2 * size_t(na) * smax) * 8 + 64));
    auto G1 = [&](int side, int a) { return wk + (0 * 2 + side) * gsum + goff[a]; };
    auto U0 = [&](int side, int a) { return wk + (1 * 2 + side) * gsum + goff[a]; };
    auto G2 = [&](int side, int a) { return wk + (2 * 2 + side) * gsum + goff[a]; };
    auto W = [&](int side, int a) { return wk + (3 * 2 + side) * gsum + goff[a]; };
    auto UF = [&](int side, int a) { return wk + (4 * 2 + side) * gsum + goff[a]; };
    double* sig = wk + 10 * gsum;
    int* ordr = static_cast<int*>(scr.get(7, (2 * size_t(na) * smax + 2 * size_t(na)) * sizeof(int)));
    int* rk = ordr + 2 * size_t(na) * smax;

    tr.mark("transpose");
    std::vector<int> kf(na);
    if (!use_jacobi_bases()) {
      // Bases by randomized rank-revealing QR (the interpolative-decomposition route;
      // the reference takes the truncated SVD of every block row, hbs.cpp:33-57):
      // 3. sketches Y = A Omega (s x l, l = min(nX, s + 16)) of the node's block row
      //    (rows side: X(f,:), the diagonal block zeroed) and block column (XT(f,:));
      // 4. Householder QR with column pivoting of Y: Q's leading columns span A's
      //    column space and |R_ii| reveals its eps-rank (#{|R_ii| > eps |R_00|}, the
      //    same relative cut as svd_rank's sigma_i > eps sigma_0).
      int lmax = 0;
      for (int a = 0; a < na; ++a) lmax = std::max(lmax, int(std::min<int64_t>(nX, ssize[slots[act[a]]] + 16)));
      double* Om = static_cast<double*>(scr.get(8, (size_t(ldX) * lmax + 2) * 8));
      double* qst = static_cast<double*>(scr.get(10, (4 * size_t(na) + 2) * 8));
      double* d_eps = qst + 4 * size_t(na);
      HLK(launch_fill_uniform(Om, int(ldX), int(nX), lmax, 0x5eed + r, st));
      HCK(cudaMemcpyAsync(d_eps, &eps, sizeof(double), cudaMemcpyHostToDevice, st));
      // The active nodes' block rows are row slices of X (block columns: of XT), all
      // sketched by the same Omega: per side ONE product Y = X Omega (nX x lmax, node a
      // uses its first l_a columns), split along K so the long reductions (K = nX) fill
      // the GPU, the K-slices summed afterwards.
      const int64_t ldY = align2(nX);
      const size_t side_sz = size_t(ldY) * lmax, slab = 2 * side_sz;
      const int tiles = std::max(1, gemm_tiles(int(nX), lmax));  // (nX = 0: every block row is zero)
      int S = std::max(1, std::min<int>(16, (4 * 148 + 2 * tiles - 1) / (2 * tiles)));
      while (S > 1 && nX / S < 256) --S;
      double* Yb = static_cast<double*>(scr.get(9, (size_t(S) * slab + 2) * 8));
      std::vector<GemmDesc> g;
      {
        const int64_t kc = ((nX + S - 1) / S + 15) / 16 * 16;  // slice boundaries 16-aligned (B columns)
        int sl = 0;
        for (int64_t k0 = 0; k0 < nX; k0 += kc, ++sl) {
          const int kk = int(std::min<int64_t>(kc, nX - k0));
          for (int side = 0; side < 2; ++side)
            g.push_back(GemmDesc{(side ? XT : X) + k0 * ldX, Om + k0, Yb + sl * slab + side * side_sz, int(nX), lmax,
                                 kk, int(ldX), int(ldX), int(ldY)});
        }
        S = sl;
      }
      if (lmax > 0) {
        gemm_batch(dbuf, g, 1.0, 0.0, true, st);
        if (S > 1) HLK(launch_sum_slices(Yb, (long long)slab, S, (long long)slab, st));
      }
      std::vector<QrDesc> q;
      for (int a = 0; a < na; ++a) {
        const int i = act[a], s = ssize[slots[i]];
        const int l = int(std::min<int64_t>(nX, s + 16)), nq = std::min(s, l);
        double* y0 = Yb + off[i];
        double* y1 = Yb + side_sz + off[i];
        q.push_back(QrDesc{y0, UF(0, a), qst + 4 * a, nullptr, int(ldY), int(align2(s)), s, nq, l - nq, 0, 0, 0});
        q.push_back(QrDesc{y1, UF(1, a), qst + 4 * a + 2, nullptr, int(ldY), int(align2(s)), s, nq, l - nq, 0, 0, 0});
      }
      QrDesc* dq = upload(dbuf, q, st);
      HLK(launch_hqr(dq, int(q.size()), smax, lmax, d_eps, st, true));
      std::vector<double> hq(4 * size_t(na));
      HCK(cudaMemcpyAsync(hq.data(), qst, hq.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      // basis columns in QR order: ordr = identity
      std::vector<int> iota(2 * size_t(na) * smax);
      for (size_t e = 0; e < iota.size(); ++e) iota[e] = int(e % size_t(smax));
      HCK(cudaMemcpyAsync(ordr, iota.data(), iota.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      HCK(cudaStreamSynchronize(st));
      for (int a = 0; a < na; ++a) kf[a] = std::max(int(hq[4 * a]), int(hq[4 * a + 2]));
    } else {
    // 3. G1: rows X(f,:) X(f,:)^T = X(f,:) XT(:,f); columns XT(f,:) X(:,f)
    {
      std::vector<GemmDesc> g;
      for (int a = 0; a < na; ++a) {
        const int i = act[a], s = ssize[slots[i]];
        const int ld = int(align2(s));
        g.push_back(GemmDesc{X + off[i], XT + off[i] * ldX, G1(0, a), s, s, int(nX), int(ldX), int(ldX), ld});
        g.push_back(GemmDesc{XT + off[i], X + off[i] * ldX, G1(1, a), s, s, int(nX), int(ldX), int(ldX), ld});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, false, st);
    }
    tr.mark("gram1");
    // 4. Jacobi on G1 -> U0
    {
      std::vector<EigDesc> e;
      for (int a = 0; a < na; ++a) {
        const int s = ssize[slots[act[a]]], ld = int(align2(s));
        for (int side = 0; side < 2; ++side) e.push_back(EigDesc{G1(side, a), U0(side, a), s, ld, ld});
      }
      EigDesc* de = upload(dbuf, e, st);
      HLK(launch_jacobi_eig(de, int(e.size()), 30, false, 0.0, smax, st));
      HCK(cudaStreamSynchronize(st));
    }
    tr.mark("jacobi1");
    // 5. B^T = A^T U0: rows side XT(:, f) U0r (nX x s) into P1, columns side X(:, f) U0c into P2
    //    (column block a of P at offset off[i] * L)
    {
      std::vector<GemmDesc> g;
      for (int a = 0; a < na; ++a) {
        const int i = act[a], s = ssize[slots[i]], ld = int(align2(s));
        g.push_back(GemmDesc{XT + off[i] * ldX, U0(0, a), P1 + off[i] * L, int(nX), s, s, int(ldX), ld, int(L)});
        g.push_back(GemmDesc{X + off[i] * ldX, U0(1, a), P2 + off[i] * L, int(nX), s, s, int(ldX), ld, int(L)});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
    }
    tr.mark("bt_gemm");
    // 6. B = (B^T)^T (s x nX, ld align2(s)) into Q1/Q2
    std::vector<size_t> qoff(na);
    {
      size_t q = 0;
      for (int a = 0; a < na; ++a) {
        qoff[a] = q;
        q += size_t(align2(ssize[slots[act[a]]])) * size_t(nX);
      }
      if (q > qbig) throw std::logic_error("compress: B workspace overflow");
      std::vector<TransDesc> t;
      for (int a = 0; a < na; ++a) {
        const int i = act[a], s = ssize[slots[i]], ld = int(align2(s));
        t.push_back(TransDesc{P1 + off[i] * L, Q1 + qoff[a], int(L), ld, int(nX), s});
        t.push_back(TransDesc{P2 + off[i] * L, Q2 + qoff[a], int(L), ld, int(nX), s});
      }
      transpose_batch(dbuf, t, st);
    }
    tr.mark("bt_trans");
    // 7. G2 = B B^T
    {
      std::vector<GemmDesc> g;
      for (int a = 0; a < na; ++a) {
        const int i = act[a], s = ssize[slots[i]], ld = int(align2(s));
        g.push_back(GemmDesc{Q1 + qoff[a], P1 + off[i] * L, G2(0, a), s, s, int(nX), ld, int(L), ld});
        g.push_back(GemmDesc{Q2 + qoff[a], P2 + off[i] * L, G2(1, a), s, s, int(nX), ld, int(L), ld});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
    }
    tr.mark("gram2");
    // 8. Jacobi (relative) on G2 -> W, lambda on the diagonal
    {
      std::vector<EigDesc> e;
      for (int a = 0; a < na; ++a) {
        const int s = ssize[slots[act[a]]], ld = int(align2(s));
        for (int side = 0; side < 2; ++side) e.push_back(EigDesc{G2(side, a), W(side, a), s, ld, ld});
      }
      EigDesc* de = upload(dbuf, e, st);
      HLK(launch_jacobi_eig(de, int(e.size()), 30, true, (1e-2 * eps) * (1e-2 * eps), smax, st));
      HCK(cudaStreamSynchronize(st));
    }
    tr.mark("jacobi2");
    // 9. Ufull = U0 W
    {
      std::vector<GemmDesc> g;
      for (int a = 0; a < na; ++a) {
        const int s = ssize[slots[act[a]]], ld = int(align2(s));
        for (int side = 0; side < 2; ++side) g.push_back(GemmDesc{U0(side, a), W(side, a), UF(side, a), s, s, s, ld, ld, ld});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
    }
    tr.mark("ufull");
    // 10. ranks (hbs.cpp:33-40, 47-57)
    {
      std::vector<SelDesc> sd;
      for (int a = 0; a < na; ++a) {
        const int s = ssize[slots[act[a]]], ld = int(align2(s));
        for (int side = 0; side < 2; ++side) {
          const size_t j = 2 * size_t(a) + side;
          sd.push_back(SelDesc{G2(side, a), ordr + j * smax, sig + j * smax, rk + j, s, ld + 1});
        }
      }
      SelDesc* ds = upload(dbuf, sd, st);
      HLK(launch_hbs_select(ds, int(sd.size()), eps, st));
      std::vector<int> hr(2 * size_t(na));
      HCK(cudaMemcpyAsync(hr.data(), rk, hr.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
      HCK(cudaStreamSynchronize(st));
      for (int a = 0; a < na; ++a) kf[a] = std::max(hr[2 * a], hr[2 * a + 1]);
    }
    }
    tr.mark("select");
    // 11. U_f, V_f = leading kf columns (s x k, ld s)
    {
      size_t tot = 0;
      for (int a = 0; a < na; ++a) tot += 2 * size_t(align2(ssize[slots[act[a]]])) * kf[a];
      double* ub = nullptr;
      ub = arena.alloc(tot + 2);
      std::vector<GatherDesc> gd;
      size_t o = 0;
      for (int a = 0; a < na; ++a) {
        const int t = slots[act[a]], s = ssize[t], ld = int(align2(s));
        H.rank[t] = kf[a];
        H.U[t] = ub + o;
        o += size_t(ld) * kf[a];
        H.V[t] = ub + o;
        o += size_t(ld) * kf[a];
        if (kf[a] == 0) continue;
        gd.push_back(GatherDesc{UF(0, a), H.U[t], ordr + (2 * size_t(a)) * smax, ld, ld, s, kf[a]});
        gd.push_back(GatherDesc{UF(1, a), H.V[t], ordr + (2 * size_t(a) + 1) * smax, ld, ld, s, kf[a]});
      }
      if (!gd.empty()) {
        GatherDesc* dg = upload(dbuf, gd, st);
        HLK(launch_gather_cols(dg, int(gd.size()), st));
      }
    }
    tr.mark("gather");
    // 12. next reduced matrix: TT = XT blockdiag(U~) (nX x nX'), T = TT^T, X' = T blockdiag(V~)
    std::vector<int64_t> noff(slots.size());
    int64_t nX2 = 0;
    std::vector<int> apos(slots.size(), -1);
    for (int a = 0; a < na; ++a) apos[act[a]] = a;
    for (size_t i = 0; i < slots.size(); ++i) {
      noff[i] = nX2;
      nX2 += apos[i] >= 0 ? kf[apos[i]] : ssize[slots[i]];
    }
    const int64_t ldX2 = align2(std::max<int64_t>(nX2, 1));
    {
      std::vector<GemmDesc> g;
      std::vector<CopyDesc> c;
      for (size_t i = 0; i < slots.size(); ++i) {
        const int t = slots[i], s = ssize[t];
        if (apos[i] >= 0) {
          if (kf[apos[i]] > 0)
            g.push_back(GemmDesc{XT + off[i] * ldX, H.U[t], P1 + noff[i] * L, int(nX), kf[apos[i]], s, int(ldX),
                                 H.ld(t), int(L)});
        } else {
          c.push_back(CopyDesc{XT + off[i] * ldX, P1 + noff[i] * L, int(ldX), int(L), int(nX), s});
        }
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
      copy_batch(dbuf, c, st);
    }
    transpose_batch(dbuf, {TransDesc{P1, P2, int(L), int(ldX2), int(nX), int(nX2)}}, st);  // T: nX' x nX
    {
      std::vector<GemmDesc> g;
      std::vector<CopyDesc> c;
      for (size_t i = 0; i < slots.size(); ++i) {
        const int t = slots[i], s = ssize[t];
        if (apos[i] >= 0) {
          const int k = kf[apos[i]];
          if (k == 0) continue;
          g.push_back(GemmDesc{P2 + off[i] * ldX2, H.V[t], X + noff[i] * ldX2, int(nX2), k, s, int(ldX2), H.ld(t),
                               int(ldX2)});
        } else {
          c.push_back(CopyDesc{P2 + off[i] * ldX2, X + noff[i] * ldX2, int(ldX2), int(ldX2), int(nX2), s});
        }
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
      copy_batch(dbuf, c, st);
    }
    tr.mark("reduce");
    for (int a = 0; a < na; ++a) ssize[slots[act[a]]] = kf[a];
    nX = nX2;
    ldX = ldX2;
  }
  HCK(cudaStreamSynchronize(st));  // before the scratch and descriptor chunks return to the pool
  return out;
}

// ---------------------------------------------------------------------------
namespace {

// Apply layout: the sweep runs on the TRANSPOSED vectors (nrhs x columns,
// ld = align2(nrhs)), so every GEMM has the batch as its M dimension (full
// 128-row DMMA tiles at large batch) and the factors as small right-hand
// operands. Every node owns a column group of the workspace:
//   leaf t:   [ y-hat_t (kp_t) ]   (x_t is read straight from X, transposed on load)
//   parent t: [ x-hat_l (kp_l) | x-hat_r (kp_r) | y-hat_t (kp_t) ]   (root: no y-hat)
// so that each step of hbs.cpp:187-232 is ONE GEMM with a contiguous A:
//   up:    x-hat_t^T = group_t[:, :inner] V_t   (leaves: x_t^T V_t)  (into the parent's group)
//   down:  y-hat_c^T = group_t [B_t^T; U_t^T][:, cols of c]    (into child c's group)
//   leaf:  y_t       = ([x_t^T | y-hat_t^T] [D_t^T; U_t^T])^T, stored transposed
// Factors are repacked once (ranks padded to even with zero rows/columns, all
// operand columns 16-byte aligned).
void pack_for_apply(HbsDev& H, cudaStream_t st) {
  auto& P = H.pk;
  if (P.ready) return;
  const int nn = int(H.nodes.size());
  P.kp.assign(nn, 0);
  P.inner.assign(nn, 0);
  P.go.assign(nn, 0);
  P.gw.assign(nn, 0);
  P.pb.assign(nn, 0);
  P.V.assign(nn, nullptr);
  P.W.assign(nn, nullptr);
  P.ldV.assign(nn, 0);
  P.ldW.assign(nn, 0);
  for (int t = 1; t < nn; ++t) P.kp[t] = int(align2(H.rank[t]));
  int64_t cols = 0, outc = 0;
  for (int t = 0; t < nn; ++t) {
    if (H.is_leaf(t)) {
      P.inner[t] = int((H.node_size(t) + 15) & ~int64_t(15));  // x columns read from X (ka, multiple of 16)
      P.pb[t] = int(outc);
      outc += align2(H.node_size(t));
    } else {
      P.inner[t] = P.kp[H.nodes[t].left] + P.kp[H.nodes[t].right];
    }
    P.gw[t] = H.is_leaf(t) ? P.kp[t] : P.inner[t] + P.kp[t];  // leaves: x is read from X itself
    P.go[t] = int(cols);
    cols += P.gw[t];
  }
  P.cols = std::max<int64_t>(cols, 2);
  P.out_cols = std::max<int64_t>(outc, 2);
  size_t tot = 0;
  for (int t = 0; t < nn; ++t) {
    const int64_t in = P.inner[t], li = std::max<int64_t>(in, 2), lw = std::max<int64_t>(in + P.kp[t], 2);
    const int64_t ncol = H.is_leaf(t) ? H.node_size(t) : in;
    if (t != 0) tot += size_t(li) * P.kp[t];  // V
    tot += size_t(lw) * ncol;                 // W
  }
  pmalloc(&P.buf, tot * 8 + 64);
  HCK(cudaMemsetAsync(P.buf, 0, tot * 8 + 64, st));
  double* base = static_cast<double*>(P.buf);
  size_t o = 0;
  std::vector<PackDesc> pd;
  for (int t = 0; t < nn; ++t) {
    const bool leaf = H.is_leaf(t);
    // inner index map (rows of V / U^T columns / B): i < i1 -> i; ip1 <= i < ip1 + i2 -> i1 + (i - ip1)
    int i1, ip1, i2;
    if (leaf) {
      i1 = int(H.node_size(t));
      ip1 = i1;
      i2 = 0;
    } else {
      const int l = H.nodes[t].left, r = H.nodes[t].right;
      i1 = H.rank[l];
      ip1 = P.kp[l];
      i2 = H.rank[r];
    }
    const int in = P.inner[t], li = std::max(in, 2), lsrc = std::max(H.ld(t), 2);
    const int k = t ? H.rank[t] : 0, kp = P.kp[t];
    const int ncol = leaf ? int(H.node_size(t)) : in;  // columns of W (= rows of D, or inner)
    if (t != 0) {
      P.V[t] = base + o;
      P.ldV[t] = li;
      o += size_t(li) * kp;
      pd.push_back(PackDesc{H.V[t], P.V[t], lsrc, li, in, kp, i1, ip1, i2, k, kp, 0, 0});
    }
    const int lw = std::max(in + kp, 2);  // W rows: [D^T or B^T (inner); U^T (kp)]
    P.W[t] = base + o;
    P.ldW[t] = lw;
    o += size_t(lw) * ncol;
    if (leaf)  // D^T in rows [0, s), the pad row stays zero
      pd.push_back(PackDesc{H.D[t], P.W[t], lsrc, lw, in, ncol, i1, ip1, 0, ncol, ncol, 0, 1});
    else  // B^T (inner x inner, the inner map on both sides)
      pd.push_back(PackDesc{H.B[t], P.W[t], lsrc, lw, in, in, i1, ip1, i2, i1, ip1, i2, 1});
    if (t != 0)  // U^T in rows [inner, inner + kp): dst(i, j) = U(map(j), i)
      pd.push_back(PackDesc{H.U[t], P.W[t] + in, lsrc, lw, kp, ncol, k, kp, 0, i1, leaf ? ncol : ip1,
                            leaf ? 0 : i2, 1});
  }
  DevBuf dbuf;
  std::vector<PackDesc> pk2;
  for (const auto& d : pd)
    if (d.rp > 0 && d.cp > 0) pk2.push_back(d);
  if (!pk2.empty()) {
    PackDesc* dd = upload(dbuf, pk2, st);
    HLK(launch_pack(dd, int(pk2.size()), st));
  }
  HCK(cudaStreamSynchronize(st));
  P.ready = true;
}

}  // namespace

// One upload of every descriptor of the call, then the whole sweep as a
// chain of batched launches on the stream with no host synchronisation.
void hbs_apply(HbsDev& H, const double* dX, int64_t ldx, int64_t nrhs, double* dY, int64_t ldy, cudaStream_t st,
               bool allow_graph) {
  if (nrhs <= 0) return;
  const int nn = int(H.nodes.size());
  DevBuf dbuf;
  if (nn == 1) {
    // Y = D X (the dense single-node case); B operand alignment: stage X
    const int64_t M = H.M, ld = align2(M);
    double* xs = nullptr;
    pmalloc(&xs, size_t(ld) * nrhs * 8 + 8);
    copy_batch(dbuf, {CopyDesc{dX, xs, int(ldx), int(ld), int(M), int(nrhs)}}, st);
    gemm_batch(dbuf, {GemmDesc{H.D[0], xs, dY, int(M), int(nrhs), int(M), H.ld(0), int(ld), int(ldy)}}, 1.0, 0.0,
               true, st);
    HCK(cudaStreamSynchronize(st));  // before the staging and descriptors return to the pool
    pool_free(xs);
    return;
  }
  pack_for_apply(H, st);
  auto& P = H.pk;
  const int64_t ldw = align2(nrhs);
  const size_t need = size_t(ldw) * size_t(P.cols);
  if (need > H.ws_doubles || ldw != H.ws_ld) {
    if (H.ws) pool_free(H.ws);
    H.ws = nullptr;
    H.ws_doubles = 0;
    pmalloc(&H.ws, need * 8 + 64);
    // zero once: the pad columns of odd-sized leaves are read (times a zero
    // factor row) but never written
    HCK(cudaMemsetAsync(H.ws, 0, need * 8 + 64, st));
    H.ws_doubles = need;
    H.ws_ld = ldw;
  }
  const int L = int(ldw);
  double* gws = H.ws;  // the node groups (ldw x cols)
  auto col = [&](int64_t c) { return gws + size_t(c) * L; };
  auto xhat_slot = [&](int c) {  // x-hat_c lives in its parent's group
    const int p = H.nodes[c].parent;
    return P.go[p] + (H.nodes[p].left == c ? 0 : P.kp[H.nodes[p].left]);
  };

  auto yhat_slot = [&](int c) { return P.go[c] + (H.is_leaf(c) ? 0 : P.inner[c]); };

  struct Phase {
    int kind;  // 0 GEMM, 3 GEMM with C stored transposed, 4 two-source GEMM, 5 two-source with C transposed
    size_t off;
    int count, tiles;
    int kmax;
  };
  std::vector<GemmDesc> gd;
  std::vector<GemmDesc2> gd2;
  std::vector<Phase> ph;
  auto add_gemm = [&](std::vector<GemmDesc>&& v, int kind = 0) {
    int tiles = 0, kmax = 0;
    std::vector<GemmDesc> keep;
    for (const auto& d : v)
      if (d.m > 0 && d.n > 0 && d.k > 0) {
        keep.push_back(d);
        tiles = std::max(tiles, gemm_tiles(d.m, d.n));
        kmax = std::max(kmax, d.k);
      }
    if (keep.empty()) return;
    ph.push_back(Phase{kind, gd.size(), int(keep.size()), tiles, kmax});
    gd.insert(gd.end(), keep.begin(), keep.end());
  };
  auto add_gemm2 = [&](std::vector<GemmDesc2>&& v, int kind) {
    int tiles = 0;
    std::vector<GemmDesc2> keep;
    for (const auto& d : v)
      if (d.m > 0 && d.n > 0 && d.k > 0) {
        keep.push_back(d);
        tiles = std::max(tiles, gemm_tiles(d.m, d.n));
      }
    if (keep.empty()) return;
    ph.push_back(Phase{kind, gd2.size(), int(keep.size()), tiles, 0});
    gd2.insert(gd2.end(), keep.begin(), keep.end());
  };
  const int R = H.height[0];
  // upward: x-hat_t^T = group_t[:, :inner] V_t; leaves: x_t^T V_t with x_t read
  // transposed straight from X (no transpose pass)
  for (int r = 0; r < R; ++r) {
    std::vector<GemmDesc> g;
    std::vector<GemmDesc2> g2;
    for (int t = 1; t < nn; ++t) {
      if (H.height[t] != r || P.kp[t] == 0) continue;
      if (H.is_leaf(t)) {
        const int s = int(H.node_size(t)), xin = P.inner[t];
        g2.push_back(GemmDesc2{dX + H.nodes[t].begin, nullptr, P.V[t], col(xhat_slot(t)), int(nrhs), P.kp[t], xin,
                               int(ldx), 0, xin, s, P.ldV[t], L});
      } else {
        g.push_back(GemmDesc{col(P.go[t]), P.V[t], col(xhat_slot(t)), int(nrhs), P.kp[t], P.inner[t], L, P.ldV[t],
                             L});
      }
    }
    add_gemm2(std::move(g2), 4);
    add_gemm(std::move(g));
  }
  // downward: y-hat_c^T = group_t [B_t^T; U_t^T][:, cols of c], one GEMM per child
  for (int r = R; r >= 1; --r) {
    std::vector<GemmDesc> g;
    for (int t = 0; t < nn; ++t) {
      if (H.height[t] != r || H.is_leaf(t)) continue;
      const int l = H.nodes[t].left, rr = H.nodes[t].right;
      const int K = P.gw[t];
      if (P.inner[t] == 0) continue;
      if (P.kp[l] > 0)
        g.push_back(GemmDesc{col(P.go[t]), P.W[t], col(yhat_slot(l)), int(nrhs), P.kp[l], K, L, P.ldW[t], L});
      if (P.kp[rr] > 0)
        g.push_back(GemmDesc{col(P.go[t]), P.W[t] + size_t(P.kp[l]) * P.ldW[t], col(yhat_slot(rr)), int(nrhs),
                             P.kp[rr], K, L, P.ldW[t], L});
    }
    add_gemm(std::move(g));
  }
  // leaves: y_t = ([x_t^T | y-hat_t^T] [D_t^T; U_t^T])^T, x_t read transposed from
  // X, y stored transposed straight into Y
  {
    std::vector<GemmDesc2> g2;
    for (int n = 0; n < nn; ++n) {
      if (!H.is_leaf(n)) continue;
      const int s = int(H.node_size(n)), xin = P.inner[n];
      g2.push_back(GemmDesc2{dX + H.nodes[n].begin, col(P.go[n]), P.W[n], dY + H.nodes[n].begin, int(nrhs), s,
                             xin + P.kp[n], int(ldx), L, xin, s, P.ldW[n], int(ldy)});
    }
    add_gemm2(std::move(g2), 5);
  }
  // one upload (both descriptor kinds), then the launches
  const size_t gbytes = gd.size() * sizeof(GemmDesc), g2bytes = gd2.size() * sizeof(GemmDesc2);
  const size_t g2_off = (gbytes + 255) & ~size_t(255);
  std::vector<unsigned char> host(g2_off + g2bytes);
  if (gbytes) std::memcpy(host.data(), gd.data(), gbytes);
  if (g2bytes) std::memcpy(host.data() + g2_off, gd2.data(), g2bytes);
  if (host.size() > H.desc_bytes) {
    if (H.d_desc) pool_free(H.d_desc);
    H.d_desc = nullptr;
    H.desc_bytes = 0;
    pmalloc(&H.d_desc, host.size());
    H.desc_bytes = host.size();
  }
  HCK(cudaMemcpyAsync(H.d_desc, host.data(), host.size(), cudaMemcpyHostToDevice, st));
  const GemmDesc* dg = static_cast<const GemmDesc*>(H.d_desc);
  const GemmDesc2* dg2 = reinterpret_cast<const GemmDesc2*>(static_cast<unsigned char*>(H.d_desc) + g2_off);
  auto launch_all = [&](cudaStream_t s2) {
    for (const Phase& f : ph) {
      if (f.kind == 4 || f.kind == 5) HLK(launch_gemm_desc2(dg2 + f.off, f.count, f.tiles, f.kind == 5, s2));
      else if (f.kind == 3) HLK(launch_gemm_desc_tc(dg + f.off, f.count, f.tiles, f.kmax, 1.0, 0.0, s2));
      else  // 128 x 64 tiles: the short reductions (K = leaf or rank) measured 20 % faster than 128 x 128
        HLK(launch_gemm_desc(dg + f.off, f.count, f.tiles, f.kmax, 1.0, 0.0, s2, true, false));
    }
  };
  // the launch sequence depends only on the tree, the ranks and nrhs: replay it as a
  // graph (one launch instead of ~16) once captured for this batch size
  static const bool graphs = std::getenv("DTN_HBS_NO_GRAPH") == nullptr;
  if (graphs && allow_graph && st != nullptr) {
    if (!(H.apply_graph && H.apply_graph_nrhs == nrhs && H.apply_graph_desc == H.d_desc)) {
      if (H.apply_graph) cudaGraphExecDestroy(H.apply_graph);
      H.apply_graph = nullptr;
      cudaGraph_t g = nullptr;
      // captured on a private stream (nothing executes during capture; the caller's
      // stream may be the legacy default stream, which cannot be captured)
      cudaStream_t cap = nullptr;
      HCK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      struct CapGuard {
        cudaStream_t s;
        ~CapGuard() { cudaStreamDestroy(s); }
      } cap_guard{cap};
      HCK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      try {
        launch_all(cap);
      } catch (...) {
        cudaStreamEndCapture(cap, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      HCK(cudaStreamEndCapture(cap, &g));
      const cudaError_t e = cudaGraphInstantiate(&H.apply_graph, g, 0);
      cudaGraphDestroy(g);
      HCK(e);
      H.apply_graph_nrhs = nrhs;
      H.apply_graph_desc = H.d_desc;
    }
    HCK(cudaGraphLaunch(H.apply_graph, st));
  } else {
    launch_all(st);
  }
  // the descriptor buffer is reused by the next call on this stream (stream order);
  // the host copy above is staged before cudaMemcpyAsync returns (pageable source)
}

// ---------------------------------------------------------------------------
namespace {

const char kMagic[8] = {'D', 'T', 'N', 'H', 'B', 'S', '0', '1'};


struct Reader {
  const uint8_t* p;
  const uint8_t* end;
  int64_t i64() {
    if (end - p < 8) throw std::invalid_argument("deserialize: truncated input");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    p += 8;
    return int64_t(v);
  }
};

}  // namespace

namespace {
struct SerMat {
  const double* d;
  int64_t ld, r, c;
};
// the DTNHBS01 matrix records in file order (hbs.cpp:446-470): per node, D (leaves),
// U and V (non-root), B (parents)
std::vector<SerMat> serial_mats(const HbsDev& H) {
  std::vector<SerMat> mats;
  for (int t = 0; t < int(H.nodes.size()); ++t) {
    const bool leaf = H.is_leaf(t);
    if (leaf) mats.push_back({H.D[t], H.ld(t), H.node_size(t), H.node_size(t)});
    if (t != 0) {
      mats.push_back({H.U[t], H.ld(t), H.rows[t], H.rank[t]});
      mats.push_back({H.V[t], H.ld(t), H.rows[t], H.rank[t]});
    }
    if (!leaf) mats.push_back({H.B[t], H.ld(t), H.rows[t], H.rows[t]});
  }
  return mats;
}
size_t serial_prefix(const HbsDev& H) { return 8 + 3 * 8 + H.nodes.size() * 6 * 8; }
}  // namespace

uint64_t hbs_serialized_size(const HbsDev& H) {
  uint64_t n = serial_prefix(H);
  for (const SerMat& x : serial_mats(H)) n += 16 + uint64_t(x.r) * uint64_t(x.c) * 8;
  return n;
}

// Every factor is packed on the device into the byte image of the record stream
// (one batched copy kernel), the image comes back in ONE device-to-host copy
// straight into the caller's buffer, and the host writes only the headers.
void hbs_serialize_into(const HbsDev& H, uint8_t* buf, cudaStream_t st) {
  const std::vector<SerMat> mats = serial_mats(H);
  const size_t prefix = serial_prefix(H);
  size_t body = 0;  // bytes after the prefix: per matrix 16 header bytes + payload
  for (const SerMat& x : mats) body += 16 + size_t(x.r) * size_t(x.c) * 8;
  DevBuf img_buf, desc_buf;  // the per-device caching pool
  double* img = static_cast<double*>(img_buf.get(std::max<size_t>(body, 8)));
  std::vector<CopyDesc> cp;
  size_t at = 0;  // in doubles, relative to the image
  for (const SerMat& x : mats) {
    at += 2;  // the (rows, cols) header
    if (x.r > 0 && x.c > 0) cp.push_back(CopyDesc{x.d, img + at, int(x.ld), int(x.r), int(x.r), int(x.c)});
    at += size_t(x.r) * size_t(x.c);
  }
  if (!cp.empty()) {
    CopyDesc* dd = upload(desc_buf, cp, st);
    HLK(launch_copy2d_batched(dd, int(cp.size()), st));
  }
  if (body) HCK(cudaMemcpyAsync(buf + prefix, img, body, cudaMemcpyDeviceToHost, st));
  // the prefix and the record headers while the copy runs
  auto put = [](uint8_t* p, int64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = uint8_t(uint64_t(v) >> (8 * i));
  };
  std::memcpy(buf, kMagic, 8);
  put(buf + 8, H.M);
  put(buf + 16, int64_t(H.nodes.size()));
  put(buf + 24, H.depth);
  uint8_t* q = buf + 32;
  for (const auto& n : H.nodes) {
    for (int64_t v : {n.begin, n.end, int64_t(n.left), int64_t(n.right), int64_t(n.parent), int64_t(n.level)}) {
      put(q, v);
      q += 8;
    }
  }
  HCK(cudaStreamSynchronize(st));
  uint8_t* h = buf + prefix;
  for (const SerMat& x : mats) {
    put(h, x.r);
    put(h + 8, x.c);
    h += 16 + size_t(x.r) * size_t(x.c) * 8;
  }
}

std::vector<uint8_t> hbs_serialize(const HbsDev& H, cudaStream_t st) {
  std::vector<uint8_t> out(hbs_serialized_size(H));
  hbs_serialize_into(H, out.data(), st);
  return out;
}

std::unique_ptr<HbsDev> hbs_deserialize(const uint8_t* data, size_t size, cudaStream_t st) {
  if (size < 8 || std::memcmp(data, kMagic, 8) != 0) throw std::invalid_argument("deserialize: bad magic");
  Reader rd{data + 8, data + size};
  auto out = std::make_unique<HbsDev>();
  HbsDev& H = *out;
  HCK(cudaGetDevice(&H.device));
  H.M = rd.i64();
  const int64_t nn = rd.i64();
  H.depth = int(rd.i64());
  if (nn < 1 || nn > (int64_t(1) << 24)) throw std::invalid_argument("deserialize: bad header");
  H.nodes.resize(size_t(nn));
  for (auto& n : H.nodes) {
    n.begin = rd.i64();
    n.end = rd.i64();
    n.left = int(rd.i64());
    n.right = int(rd.i64());
    n.parent = int(rd.i64());
    n.level = int(rd.i64());
  }
  if (H.nodes[0].end != H.M || H.nodes[0].begin != 0) throw std::invalid_argument("deserialize: bad header");
  hbs_check_tree(H.nodes, H.M, "deserialize");
  H.rank.assign(nn, 0);
  H.rows.assign(nn, 0);
  H.height.assign(nn, 0);
  H.D.assign(nn, nullptr);
  H.U.assign(nn, nullptr);
  H.V.assign(nn, nullptr);
  H.B.assign(nn, nullptr);
  for (int t = int(nn) - 1; t >= 0; --t)
    if (!H.is_leaf(t)) H.height[t] = 1 + std::max(H.height[H.nodes[t].left], H.height[H.nodes[t].right]);
  // first pass: shapes
  struct Mat {
    int64_t r, c;
    const uint8_t* p;
  };
  std::vector<Mat> mats;
  size_t total = 0;
  auto matrix = [&]() {
    const int64_t r = rd.i64(), c = rd.i64();
    if (r < 0 || c < 0) throw std::invalid_argument("deserialize: bad matrix shape");
    const size_t bytes = size_t(r) * size_t(c) * 8;
    if (size_t(rd.end - rd.p) < bytes) throw std::invalid_argument("deserialize: truncated input");
    mats.push_back({r, c, rd.p});
    rd.p += bytes;
    total += size_t(align2(r)) * size_t(c);
  };
  for (int t = 0; t < int(nn); ++t) {
    const bool leaf = H.is_leaf(t);
    if (leaf) matrix();
    if (t != 0) {
      matrix();
      matrix();
    }
    if (!leaf) matrix();
  }
  {  // every factor's shape against the tree (hbs.hpp:30-51) before anything reaches the device:
     // leaf D s x s; U, V rows x rank (equal shapes; rows = s on leaves, k_left + k_right on
     // parents); parent B (k_left + k_right)^2
    std::vector<int64_t> rk(size_t(nn), 0), rw(size_t(nn), 0);
    size_t mi = 0;
    std::vector<size_t> first(static_cast<size_t>(nn), 0);
    for (int t = 0; t < int(nn); ++t) {
      first[size_t(t)] = mi;
      mi += (H.is_leaf(t) ? 1 : 0) + (t != 0 ? 2 : 0) + (H.is_leaf(t) ? 0 : 1);
    }
    for (int t = int(nn) - 1; t >= 0; --t) {  // children before parents (preorder: children have larger ids)
      const auto& n = H.nodes[t];
      size_t q = first[size_t(t)];
      const int64_t s = n.end - n.begin;
      int64_t rows = s;
      if (H.is_leaf(t)) {
        const Mat& d = mats[q++];
        if (d.r != s || d.c != s) throw std::invalid_argument("deserialize: leaf D shape does not match the tree");
      } else {
        rows = rk[size_t(n.left)] + rk[size_t(n.right)];
      }
      rw[size_t(t)] = rows;
      if (t != 0) {
        const Mat& u = mats[q++];
        const Mat& v = mats[q++];
        if (u.r != rows || v.r != rows || u.c != v.c || u.c > rows)
          throw std::invalid_argument("deserialize: U/V shape does not match the tree");
        rk[size_t(t)] = u.c;
      }
      if (!H.is_leaf(t)) {
        const Mat& b = mats[q++];
        if (b.r != rows || b.c != rows) throw std::invalid_argument("deserialize: B shape does not match the tree");
      }
    }
  }
  double* buf = nullptr;
  pmalloc(&buf, total * 8 + 8);
  H.buffers.push_back(buf);
  size_t o = 0, m = 0;
  auto place = [&](double*& dst) {
    const Mat& x = mats[m++];
    dst = buf + o;
    const int64_t ld = align2(x.r);
    if (x.r > 0 && x.c > 0)
      HCK(cudaMemcpy2D(dst, size_t(ld) * 8, x.p, size_t(x.r) * 8, size_t(x.r) * 8, size_t(x.c), cudaMemcpyHostToDevice));
    o += size_t(ld) * size_t(x.c);
    return x;
  };
  for (int t = 0; t < int(nn); ++t) {
    const bool leaf = H.is_leaf(t);
    if (leaf) {
      const Mat x = place(H.D[t]);
      H.rows[t] = int(x.r);
    }
    if (t != 0) {
      const Mat u = place(H.U[t]);
      place(H.V[t]);
      H.rank[t] = int(u.c);
      H.rows[t] = int(u.r);
    }
    if (!leaf) {
      const Mat b = place(H.B[t]);
      H.rows[t] = int(b.r);
    }
  }
  (void)st;
  return out;
}

// ---------------------------------------------------------------------------
// invert_hbs (hbs_ops.cpp:148-201), one tree height at a time, every node of
// that height in the same batched launches. Per non-root node t (s = rows[t],
// k = rank[t]):
//   Dtilde = D_t (leaf) or B_t + diag(Dhat_left, Dhat_right)   add_blocks
//   Dinv   = Dtilde^{-1}                                        gj_inverse
//   W = Dinv U,  VT = V^T,  Dhat = (VT W)^{-1}                  GEMM, transpose, gj_inverse
//   E = W Dhat,  Z = VT Dinv,  F = (Dhat Z)^T                   GEMM, transpose
//   G = Dinv - E Z                                              copy + GEMM (C -= A B)
// (F = Dinv^T V Dhat^T and G = Dinv - E V^T Dinv exactly as the reference
// writes them); the root's core inverse is (B_0 + diag(Dhat_l, Dhat_r))^{-1}.
// Eigen's FullPivLU inverses become partial-pivoting Gauss-Jordan inverses
// (same result to rounding on invertible blocks); a zero or non-finite pivot
// raises HbsSingular with the reference's "what [node t level l]" text.
std::unique_ptr<HbsDev> hbs_invert(const HbsDev& H, cudaStream_t st) {
  auto out = std::make_unique<HbsDev>();
  HbsDev& R = *out;
  R.device = H.device;
  R.M = H.M;
  R.depth = H.depth;
  R.nodes = H.nodes;
  R.rank = H.rank;
  R.rows = H.rows;
  R.height = H.height;
  const int nn = int(H.nodes.size());
  R.D.assign(nn, nullptr);
  R.U.assign(nn, nullptr);
  R.V.assign(nn, nullptr);
  R.B.assign(nn, nullptr);
  DevBuf dbuf, ibuf;
  struct Frees {
    std::vector<void*> v;
    ~Frees() {
      for (void* p : v) pool_free(p);
    }
  } frees;
  // all factor storage in one allocation, per-level work in one reused buffer
  size_t keep_all = 0, work_max = 0, dhat_all = 0;
  {
    std::vector<size_t> keep_h(64, 0), work_h(64, 0);
    for (int t = 0; t < nn; ++t) {
      const size_t s = size_t(H.rows[t]), k = size_t(H.rank[t]), ls = size_t(align2(s));
      const size_t lk = size_t(std::max<int64_t>(align2(k), 2));
      const int h = std::min(H.height[t], 63);
      keep_h[h] += ls * s + (t ? 2 * ls * k : 0) + 8;
      work_h[h] += ls * s + (t ? ls * k + 3 * lk * s : 0) + 8;
      if (t) dhat_all += size_t(align2(k)) * k + 2;
    }
    for (int h = 0; h < 64; ++h) {
      keep_all += keep_h[h];
      work_max = std::max(work_max, work_h[h]);
    }
  }
  Arena arena(R, keep_all + 64);
  double* work_buf = nullptr;
  pmalloc(&work_buf, (work_max + dhat_all + 64) * 8);
  frees.v.push_back(work_buf);
  bool dhat_taken = false;
  auto dalloc = [&](size_t doubles, bool keep) {
    if (keep) return arena.alloc(doubles);
    // the Dhat block (first request) sits after the per-level work area
    if (!dhat_taken) {
      dhat_taken = true;
      return work_buf + work_max + 2;
    }
    return work_buf;
  };
  int* dinfo = nullptr;
  pmalloc(&dinfo, 2 * size_t(nn) * sizeof(int) + 16);  // every node inverts at most two blocks
  frees.v.push_back(dinfo);
  auto where = [&](int t) {
    return "node " + std::to_string(t) + " level " + std::to_string(H.nodes[t].level);
  };
  // batched in-place inverses, their singularity flags checked once at the end (no
  // synchronisation per level): the error names the first failing batch in program
  // order and its singular block with the lowest node id, as a per-batch check would
  struct InvCall {
    std::vector<int> nodes;
    size_t slot0;
    const char* what;
  };
  std::vector<InvCall> calls;
  size_t nslots = 0;
  auto invert = [&](const std::vector<std::pair<int, InvDesc>>& blocks, const char* what) {
    if (blocks.empty()) return;
    std::vector<InvDesc> v;
    int smax = 0;
    InvCall call{{}, nslots, what};
    for (size_t i = 0; i < blocks.size(); ++i) {
      InvDesc d = blocks[i].second;
      d.info = dinfo + nslots + i;
      v.push_back(d);
      smax = std::max(smax, d.s);
      call.nodes.push_back(blocks[i].first);
    }
    nslots += blocks.size();
    calls.push_back(std::move(call));
    InvDesc* dv = upload(ibuf, v, st);
    HLK(launch_gj_inverse(dv, int(v.size()), smax, st));
  };
  auto check_singular = [&]() {
    std::vector<int> info(nslots);
    if (nslots) HCK(cudaMemcpyAsync(info.data(), dinfo, nslots * sizeof(int), cudaMemcpyDeviceToHost, st));
    HCK(cudaStreamSynchronize(st));
    for (const InvCall& c : calls) {
      int bad = -1;
      for (size_t i = 0; i < c.nodes.size(); ++i)
        if (info[c.slot0 + i] != 0 && (bad < 0 || c.nodes[i] < bad)) bad = c.nodes[i];
      if (bad >= 0) throw HbsSingular(std::string(c.what) + " is singular [" + where(bad) + "]");
    }
  };

  if (nn == 1) {  // hbs_ops.cpp:157-160
    const int s = int(H.M), ld = H.ld(0);
    R.D[0] = dalloc(size_t(ld) * s, true);
    copy_batch(dbuf, {CopyDesc{H.D[0], R.D[0], ld, ld, s, s}}, st);
    invert({{0, InvDesc{R.D[0], nullptr, s, ld}}}, "D");
    try {
      check_singular();
    } catch (const HbsSingular&) {
      throw HbsSingular("D is singular [root leaf]");
    }
    return out;
  }

  // Dhat_t (k x k, ld align2(k)) of every non-root node, kept until its parent is done
  std::vector<double*> dhat(nn, nullptr);
  {
    size_t tot = 0;
    for (int t = 1; t < nn; ++t) tot += size_t(align2(H.rank[t])) * H.rank[t];
    double* base = dalloc(tot, false);
    size_t o = 0;
    for (int t = 1; t < nn; ++t) {
      dhat[t] = base + o;
      o += size_t(align2(H.rank[t])) * H.rank[t];
    }
  }
  const int RH = H.height[0];
  for (int r = 0; r <= RH; ++r) {
    std::vector<int> act;
    for (int t = 0; t < nn; ++t)
      if (H.height[t] == r) act.push_back(t);
    if (act.empty()) continue;
    // storage: result factors (kept) and per-level work
    size_t keep = 0, work = 0;
    for (int t : act) {
      const size_t s = size_t(H.rows[t]), k = size_t(H.rank[t]), ls = size_t(align2(s));
      const size_t lk = size_t(std::max<int64_t>(align2(k), 2));
      keep += ls * s + (t ? 2 * ls * k : 0);
      work += ls * s + (t ? ls * k + 3 * lk * s : 0);
    }
    double* kb = dalloc(keep, true);
    double* wb = dalloc(work, false);
    struct Slot {
      double *Dt = nullptr, *W = nullptr, *VT = nullptr, *Z = nullptr, *FT = nullptr;
    };
    std::vector<Slot> sl(nn);
    size_t ko = 0, wo = 0;
    for (int t : act) {
      const size_t s = size_t(H.rows[t]), k = size_t(H.rank[t]), ls = size_t(align2(s));
      const size_t lk = size_t(std::max<int64_t>(align2(k), 2));
      (H.is_leaf(t) ? R.D[t] : R.B[t]) = kb + ko;
      ko += ls * s;
      Slot& q = sl[t];
      q.Dt = wb + wo;
      wo += ls * s;
      if (t) {
        R.U[t] = kb + ko;
        ko += ls * k;
        R.V[t] = kb + ko;
        ko += ls * k;
        q.W = wb + wo;
        wo += ls * k;
        q.VT = wb + wo;
        wo += lk * s;
        q.Z = wb + wo;
        wo += lk * s;
        q.FT = wb + wo;
        wo += lk * s;
      }
    }
    // 1. Dtilde
    {
      std::vector<CopyDesc> c;
      std::vector<AddDesc> a;
      for (int t : act) {
        const int s = H.rows[t], ld = H.ld(t);
        if (s == 0) continue;
        c.push_back(CopyDesc{H.is_leaf(t) ? H.D[t] : H.B[t], sl[t].Dt, ld, ld, s, s});
        if (!H.is_leaf(t)) {
          const int l = H.nodes[t].left, rr = H.nodes[t].right, k1 = H.rank[l], k2 = H.rank[rr];
          if (k1) a.push_back(AddDesc{dhat[l], sl[t].Dt, int(align2(k1)), ld, k1, k1});
          if (k2) a.push_back(AddDesc{dhat[rr], sl[t].Dt + k1 + size_t(k1) * ld, int(align2(k2)), ld, k2, k2});
        }
      }
      copy_batch(dbuf, c, st);
      if (!a.empty()) {
        AddDesc* da = upload(dbuf, a, st);
        HLK(launch_add_blocks(da, int(a.size()), st));
      }
    }
    // 2. Dinv (at the root: the core inverse, hbs_ops.cpp:177-180)
    {
      std::vector<std::pair<int, InvDesc>> b;
      for (int t : act)
        if (H.rows[t] > 0) b.push_back({t, InvDesc{sl[t].Dt, nullptr, H.rows[t], H.ld(t)}});
      invert(b, r == RH ? "root coupling block" : "Dtilde");
    }
    if (r == RH) {  // act = {0}
      const int s = H.rows[0], ld = H.ld(0);
      if (s > 0) copy_batch(dbuf, {CopyDesc{sl[0].Dt, R.B[0], ld, ld, s, s}}, st);
      break;
    }
    // 3. W = Dinv U, VT = V^T
    {
      std::vector<GemmDesc> g;
      std::vector<TransDesc> tr;
      for (int t : act) {
        const int s = H.rows[t], k = H.rank[t], ld = H.ld(t), lk = std::max(int(align2(k)), 2);
        if (s == 0 || k == 0) continue;
        g.push_back(GemmDesc{sl[t].Dt, H.U[t], sl[t].W, s, k, s, ld, ld, ld});
        tr.push_back(TransDesc{H.V[t], sl[t].VT, ld, lk, s, k});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
      transpose_batch(dbuf, tr, st);
    }
    // 4. T = VT W -> Dhat = T^{-1}
    {
      std::vector<GemmDesc> g;
      for (int t : act) {
        const int s = H.rows[t], k = H.rank[t], ld = H.ld(t), lk = std::max(int(align2(k)), 2);
        if (s == 0 || k == 0) continue;
        g.push_back(GemmDesc{sl[t].VT, sl[t].W, dhat[t], k, k, s, lk, ld, int(align2(k))});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
      std::vector<std::pair<int, InvDesc>> b;
      for (int t : act)
        if (H.rank[t] > 0) b.push_back({t, InvDesc{dhat[t], nullptr, H.rank[t], int(align2(H.rank[t]))}});
      invert(b, "reduced block (V^T Dtilde^{-1} U)");
    }
    // 5. E = W Dhat (U slot); Z = VT Dinv
    {
      std::vector<GemmDesc> g;
      for (int t : act) {
        const int s = H.rows[t], k = H.rank[t], ld = H.ld(t), lk = std::max(int(align2(k)), 2);
        if (s == 0 || k == 0) continue;
        g.push_back(GemmDesc{sl[t].W, dhat[t], R.U[t], s, k, k, ld, int(align2(k)), ld});
        g.push_back(GemmDesc{sl[t].VT, sl[t].Dt, sl[t].Z, k, s, s, lk, ld, lk});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
    }
    // 6. FT = Dhat Z, F = FT^T (V slot); G = Dinv - E Z (D / B slot)
    {
      std::vector<GemmDesc> g;
      std::vector<CopyDesc> c;
      for (int t : act) {
        const int s = H.rows[t], k = H.rank[t], ld = H.ld(t), lk = std::max(int(align2(k)), 2);
        if (s == 0) continue;
        c.push_back(CopyDesc{sl[t].Dt, H.is_leaf(t) ? R.D[t] : R.B[t], ld, ld, s, s});
        if (k == 0) continue;
        g.push_back(GemmDesc{dhat[t], sl[t].Z, sl[t].FT, k, s, k, int(align2(k)), lk, lk});
      }
      gemm_batch(dbuf, g, 1.0, 0.0, true, st);
      copy_batch(dbuf, c, st);
      std::vector<TransDesc> tr;
      std::vector<GemmDesc> gu;
      for (int t : act) {
        const int s = H.rows[t], k = H.rank[t], ld = H.ld(t), lk = std::max(int(align2(k)), 2);
        if (s == 0 || k == 0) continue;
        tr.push_back(TransDesc{sl[t].FT, R.V[t], lk, ld, k, s});
        gu.push_back(GemmDesc{R.U[t], sl[t].Z, H.is_leaf(t) ? R.D[t] : R.B[t], s, s, k, ld, lk, ld});
      }
      transpose_batch(dbuf, tr, st);
      gemm_batch(dbuf, gu, -1.0, 1.0, true, st);
    }
  }
  check_singular();  // (synchronises the stream)
  return out;
}

}  // namespace dtnb
