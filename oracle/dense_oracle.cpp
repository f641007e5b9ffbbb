// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by, or called
// from the product path (paper_1302_5995_b200/); only tests/, the smoke check
// in __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg use
// it, and only as the checker or the timed CPU baseline.
//
// CPU restatement of the reference's dense build path (the reference itself,
// /root/reference/proj, cannot be compiled here: it needs Eigen3, which is
// absent — proj/CMakeLists.txt:10). Each function cites the reference
// file:line it restates. Dense kernels (LU with partial pivoting, triangular
// solves, GEMM) go to the numpy-bundled OpenBLAS (ILP64, scipy_ prefix) in
// place of Eigen's PartialPivLU / SparseLU / GEMM; orderings, merge order and
// the singularity test are the reference's.
//
// Parity pins (tests/test_oracle_*.py): the reference's own formula-level
// known-answer tests — proj/tests/test_grid.cpp (stencil values, ordering,
// partition), proj/tests/test_dense_nd.cpp (hand elimination, brute-force
// Schur complement of the assembled matrix at 1e-10..1e-14, pairing order,
// symmetry, G S = I) and proj/tests/acceptance.cpp:74-114 (criterion 1, all
// catalog problems × n in {8,16,32}).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

extern "C" {
// OpenBLAS (ILP64, scipy-prefixed) shipped in numpy.libs
void scipy_dgetrf_64_(const int64_t* m, const int64_t* n, double* a, const int64_t* lda,
                      int64_t* ipiv, int64_t* info);
void scipy_dgetrs_64_(const char* trans, const int64_t* n, const int64_t* nrhs, const double* a,
                      const int64_t* lda, const int64_t* ipiv, double* b, const int64_t* ldb,
                      int64_t* info, size_t);
void scipy_dgbsv_64_(const int64_t* n, const int64_t* kl, const int64_t* ku, const int64_t* nrhs,
                     double* ab, const int64_t* ldab, int64_t* ipiv, double* b, const int64_t* ldb,
                     int64_t* info);
void scipy_dgemm_64_(const char* ta, const char* tb, const int64_t* m, const int64_t* n,
                     const int64_t* k, const double* alpha, const double* a, const int64_t* lda,
                     const double* b, const int64_t* ldb, const double* beta, double* c,
                     const int64_t* ldc, size_t, size_t);
void scipy_dtrsm_64_(const char* side, const char* uplo, const char* transa, const char* diag, const int64_t* m,
                     const int64_t* n, const double* alpha, const double* a, const int64_t* lda, double* b,
                     const int64_t* ldb, size_t, size_t, size_t, size_t);
void scipy_dlaswp_64_(const int64_t* n, double* a, const int64_t* lda, const int64_t* k1, const int64_t* k2,
                      const int64_t* ipiv, const int64_t* incx);
void scipy_openblas_set_num_threads64_(int);
int scipy_openblas_get_num_threads64_(void);
}

namespace orc {

using Index = int64_t;

struct Mat {  // column-major, like Eigen::MatrixXd
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(size_t(r) * size_t(c), 0.0) {}
  double& operator()(Index i, Index j) { return a[size_t(j) * rows + i]; }
  double operator()(Index i, Index j) const { return a[size_t(j) * rows + i]; }
};

struct FactorizationError : std::runtime_error {
  // restates dtn::FactorizationError (errors.hpp:11-21): what + " [" + where + "]"
  FactorizationError(const std::string& what, const std::string& where)
      : std::runtime_error(what + " [" + where + "]") {}
};

// ---------------------------------------------------------------- grid.hpp/cpp
struct GridPoint { int x, y; };

struct Lattice {  // grid.hpp:56-78
  int n = 0;
  int side() const { return n - 2; }
  Index num_unknowns() const { return Index(side()) * side(); }
  bool is_unknown(int x, int y) const { return x >= 1 && x <= n - 2 && y >= 1 && y <= n - 2; }
  Index unknown_id(int x, int y) const { return Index(y - 1) * side() + (x - 1); }
  GridPoint point_of(Index id) const { return {int(id % side()) + 1, int(id / side()) + 1}; }
  Index ring_id(int x, int y) const {  // grid.cpp:40-47
    const int m = n - 1;
    if (y == 0) return x;
    if (x == m) return m + y;
    if (y == m) return 2 * m + (m - x);
    if (x == 0) return 3 * m + (m - y);
    throw std::logic_error("ring_id: node is not on the outer ring");
  }
};

// Assembled 5-point operator: per unknown the center and E,W,N,S couplings
// (grid.cpp:130-160, neighbor order east, west, north, south). A coupling to
// a ring node is a Dirichlet-forcing entry, not part of A.
struct Operator {
  int n = 0;
  double h = 0.0;
  Lattice lat;
  std::vector<double> center, east, west, north, south;
  double coeff(Index row, Index col) const {  // DiscreteOperator::coeff, grid.cpp:49-55
    if (row == col) return center[row];
    const GridPoint p = lat.point_of(row), q = lat.point_of(col);
    if (q.y == p.y && q.x == p.x + 1) return east[row];
    if (q.y == p.y && q.x == p.x - 1) return west[row];
    if (q.x == p.x && q.y == p.y + 1) return north[row];
    if (q.x == p.x && q.y == p.y - 1) return south[row];
    return 0.0;
  }
};

double uniform01(std::mt19937_64& rng) { return double(rng() >> 11) * 0x1.0p-53; }  // grid.cpp:77-79

using Field = std::function<double(double, double)>;

// discretize, continuum branch (grid.cpp:106-144, 160-168)
Operator discretize_continuum(int n, const Field& b, const Field& c, const Field& d) {
  if (n < 4) throw std::invalid_argument("discretize: n must be >= 4");
  Operator op;
  op.n = n;
  op.h = 1.0 / (n - 1);
  op.lat = Lattice{n};
  const Index nu = op.lat.num_unknowns();
  for (auto* v : {&op.center, &op.east, &op.west, &op.north, &op.south}) v->assign(nu, 0.0);
  const double h = op.h;
  for (int y = 1; y <= n - 2; ++y) {
    for (int x = 1; x <= n - 2; ++x) {
      const Index row = op.lat.unknown_id(x, y);
      const double px = x * h, py = y * h;
      const double bv = b ? b(px, py) : 0.0, cv = c ? c(px, py) : 0.0, dv = d ? d(px, py) : 0.0;
      if (!std::isfinite(bv) || !std::isfinite(cv) || !std::isfinite(dv))
        throw std::domain_error("discretize: coefficient is not finite");
      const double ih2 = 1.0 / (h * h), ih = 1.0 / h;
      op.center[row] = 4.0 * ih2 + dv;
      op.east[row] = -ih2 + bv * ih;
      op.west[row] = -ih2 - bv * ih;
      op.north[row] = -ih2 + cv * ih;
      op.south[row] = -ih2 - cv * ih;
    }
  }
  return op;
}

// discretize, network branch (grid.cpp:82-92, 125-131, 145-150)
Operator discretize_network(int n, double lo, double hi, uint64_t seed) {
  if (n < 4) throw std::invalid_argument("discretize: n must be >= 4");
  Operator op;
  op.n = n;
  op.h = 1.0 / (n - 1);
  op.lat = Lattice{n};
  const Index nu = op.lat.num_unknowns();
  for (auto* v : {&op.center, &op.east, &op.west, &op.north, &op.south}) v->assign(nu, 0.0);
  std::vector<double> sigma;
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < size_t(2) * n * (n - 1); ++i) sigma.push_back(lo + (hi - lo) * uniform01(rng));
  auto sig_h = [&](int x, int y) { return sigma[size_t(y) * (n - 1) + x]; };
  auto sig_v = [&](int x, int y) { return sigma[size_t(n) * (n - 1) + size_t(y) * n + x]; };
  for (int y = 1; y <= n - 2; ++y) {
    for (int x = 1; x <= n - 2; ++x) {
      const Index row = op.lat.unknown_id(x, y);
      const double se = sig_h(x, y), sw = sig_h(x - 1, y), sn = sig_v(x, y), ss = sig_v(x, y - 1);
      op.center[row] = se + sw + sn + ss;
      op.east[row] = -se;
      op.west[row] = -sw;
      op.north[row] = -sn;
      op.south[row] = -ss;
    }
  }
  return op;
}

// discrete_eigenvalue / _kth (problems.cpp:75-110), needed by helmholtz3
double discrete_eigenvalue(int p, int q, int n) {
  const double h = 1.0 / (n - 1);
  return (4.0 - 2.0 * (std::cos(p * std::numbers::pi / (n - 1)) + std::cos(q * std::numbers::pi / (n - 1)))) / (h * h);
}
double discrete_eigenvalue_kth(int k, int n) {
  const int cap = std::min(n - 2, std::max(2 * k, 8));
  if (int64_t(cap) * cap < k) throw std::invalid_argument("discrete_eigenvalue_kth: k exceeds spectrum");
  struct E { double l; int p, q; };
  std::vector<E> es;
  for (int p = 1; p <= cap; ++p)
    for (int q = 1; q <= cap; ++q) es.push_back({discrete_eigenvalue(p, q, n), p, q});
  std::sort(es.begin(), es.end(), [](const E& a, const E& b) {
    if (a.l != b.l) return a.l < b.l;
    return std::pair(a.p, a.q) < std::pair(b.p, b.q);
  });
  return es[size_t(k) - 1].l;
}

// Catalog (problems.cpp:26-73) plus the BASELINE.json configs.
Operator make_problem(const std::string& name, int n, double param, uint64_t seed) {
  const double pi = std::numbers::pi;
  auto cst = [](double v) { return Field([v](double, double) { return v; }); };
  Field zero = cst(0.0);
  if (name == "laplace") return discretize_continuum(n, zero, zero, zero);
  if (name == "diffconv1") return discretize_continuum(n, cst(100.0), zero, zero);
  if (name == "diffconv2") return discretize_continuum(n, cst(1000.0), zero, zero);
  if (name == "diffconv3")
    return discretize_continuum(n, [=](double, double y) { return 125.0 * std::cos(4.0 * pi * y); },
                                [=](double x, double) { return 125.0 * std::sin(4.0 * pi * x); }, zero);
  if (name == "diffconv4")
    return discretize_continuum(n, [=](double x, double) { return 125.0 * std::cos(4.0 * pi * x); },
                                [=](double, double y) { return 125.0 * std::sin(4.0 * pi * y); }, zero);
  if (name == "helmholtz1") return discretize_continuum(n, zero, zero, cst(-100.0));
  if (name == "helmholtz2") return discretize_continuum(n, zero, zero, cst(-4005.0));
  if (name == "helmholtz3") return discretize_continuum(n, zero, zero, cst(-discrete_eigenvalue_kth(10, n) + 1e-5));
  if (name == "helmholtz4") {
    const double k = 2.0 * pi * n / 40.0;
    return discretize_continuum(n, zero, zero, cst(-k * k));
  }
  if (name == "random1") return discretize_network(n, 1.0, 2.0, seed);
  if (name == "random2") return discretize_network(n, 1.0, 1000.0, seed);
  // ProblemSpec::network("uniform", n, 1, 1, seed) used by test_dense_nd.cpp:72-90
  if (name == "uniform") return discretize_network(n, 1.0, 1.0, seed);
  // BASELINE.json configs (param = kappa)
  if (name == "helmholtz") return discretize_continuum(n, zero, zero, cst(-param * param));
  if (name == "varcoef") {
    const double k2 = param * param;
    return discretize_continuum(
        n, [=](double, double y) { return 50.0 * std::cos(4.0 * pi * y); },
        [=](double x, double) { return 50.0 * std::sin(4.0 * pi * x); },
        [=](double x, double y) {
          return -k2 * (1.0 - 0.5 * std::exp(-((x - 0.5) * (x - 0.5) + (y - 0.5) * (y - 0.5)) / 0.02));
        });
  }
  throw std::invalid_argument("catalog: unknown problem '" + name + "'");
}

std::vector<GridPoint> rect_perimeter_ccw(int x0, int x1, int y0, int y1) {  // grid.cpp:170-190
  std::vector<GridPoint> p;
  if (x0 > x1 || y0 > y1) return p;
  if (x0 == x1 && y0 == y1) return {{x0, y0}};
  if (x0 == x1) { for (int y = y0; y <= y1; ++y) p.push_back({x0, y}); return p; }
  if (y0 == y1) { for (int x = x0; x <= x1; ++x) p.push_back({x, y0}); return p; }
  for (int x = x0; x <= x1; ++x) p.push_back({x, y0});
  for (int y = y0 + 1; y <= y1; ++y) p.push_back({x1, y});
  for (int x = x1 - 1; x >= x0; --x) p.push_back({x, y1});
  for (int y = y1 - 1; y >= y0 + 1; --y) p.push_back({x0, y});
  return p;
}

struct GridBox {  // grid.hpp:120-141
  int id = -1, level = 0, parent = -1;
  std::array<int, 4> children{-1, -1, -1, -1};  // SW, SE, NW, NE
  int gx0 = 0, gx1 = 0, gy0 = 0, gy1 = 0;
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  std::vector<Index> interior, boundary;
};

struct BoxTree {
  int n = 0, n_leaf = 0, depth = 0;
  std::vector<GridBox> boxes;
  std::vector<std::vector<int>> levels;
};

void fill_index_sets(GridBox& box, const Lattice& lat) {  // grid.cpp:194-209
  box.x0 = std::max(box.gx0, 1);
  box.y0 = std::max(box.gy0, 1);
  box.x1 = std::min(box.gx1, lat.n - 1) - 1;
  box.y1 = std::min(box.gy1, lat.n - 1) - 1;
  if (box.x0 > box.x1 || box.y0 > box.y1) return;
  for (const auto& gp : rect_perimeter_ccw(box.x0, box.x1, box.y0, box.y1))
    box.boundary.push_back(lat.unknown_id(gp.x, gp.y));
  for (int y = box.y0 + 1; y <= box.y1 - 1; ++y)
    for (int x = box.x0 + 1; x <= box.x1 - 1; ++x) box.interior.push_back(lat.unknown_id(x, y));
}

// build_tree (grid.cpp:213-266). uniform_side > 0 selects the test-only
// uniform variant: unknown rectangles are halved exactly (requires
// n-2 == uniform_side * 2^L); the root S does not depend on the partition.
BoxTree build_tree(int n, int n_leaf, int uniform_side) {
  if (n < 4) throw std::invalid_argument("build_tree: n must be >= 4");
  BoxTree tree;
  tree.n = n;
  const Lattice lat{n};
  int depth = 0;
  if (uniform_side > 0) {
    int s = n - 2;
    while (s > uniform_side) {
      if (s % 2) throw std::invalid_argument("build_tree: n-2 is not leaf_side * 2^L");
      s /= 2;
      ++depth;
    }
    if (s != uniform_side) throw std::invalid_argument("build_tree: n-2 is not leaf_side * 2^L");
    tree.n_leaf = uniform_side * uniform_side;
  } else {
    if (n_leaf < 16) throw std::invalid_argument("build_tree: n_leaf must be >= 16");
    while (double(n) * n > double(n_leaf) * std::pow(4.0, depth)) ++depth;
    tree.n_leaf = n_leaf;
  }
  tree.depth = depth;
  tree.levels.resize(depth + 1);
  GridBox root;
  root.id = 0;
  root.gx0 = 0; root.gx1 = n; root.gy0 = 0; root.gy1 = n;
  if (uniform_side > 0) { root.gx0 = 1; root.gx1 = n - 1; root.gy0 = 1; root.gy1 = n - 1; }
  fill_index_sets(root, lat);
  tree.boxes.push_back(root);
  tree.levels[0].push_back(0);
  for (int lev = 0; lev < depth; ++lev) {
    for (int id : tree.levels[lev]) {
      const int gx0 = tree.boxes[id].gx0, gx1 = tree.boxes[id].gx1;
      const int gy0 = tree.boxes[id].gy0, gy1 = tree.boxes[id].gy1;
      int xm = gx0 + (gx1 - gx0 + 1) / 2, ym = gy0 + (gy1 - gy0 + 1) / 2;
      if (uniform_side > 0) { xm = gx0 + (gx1 - gx0) / 2; ym = gy0 + (gy1 - gy0) / 2; }
      const std::array<std::array<int, 4>, 4> regions{{{gx0, xm, gy0, ym}, {xm, gx1, gy0, ym},
                                                       {gx0, xm, ym, gy1}, {xm, gx1, ym, gy1}}};
      for (int c = 0; c < 4; ++c) {
        GridBox child;
        child.id = int(tree.boxes.size());
        child.level = lev + 1;
        child.parent = id;
        child.gx0 = regions[c][0]; child.gx1 = regions[c][1];
        child.gy0 = regions[c][2]; child.gy1 = regions[c][3];
        fill_index_sets(child, lat);
        tree.boxes[id].children[c] = child.id;
        tree.levels[lev + 1].push_back(child.id);
        tree.boxes.push_back(std::move(child));
      }
    }
  }
  return tree;
}

// ------------------------------------------------------------- dense_nd.cpp
struct SchurData {  // dense_nd.hpp:18-26
  int box_id = -1;
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  std::vector<Index> boundary;
  Mat S;
};

void gemm_sub(const Mat& A, const Mat& B, Mat& C) {  // C -= A*B
  const int64_t m = A.rows, n = B.cols, k = A.cols;
  if (m == 0 || n == 0 || k == 0) return;
  const double alpha = -1.0, beta = 1.0;
  scipy_dgemm_64_("N", "N", &m, &n, &k, &alpha, A.a.data(), &m, B.a.data(), &k, &beta, C.a.data(), &m, 1, 1);
}

// leaf_schur (dense_nd.cpp:37-103). A_ii is banded in the row-major interior
// ordering (half bandwidth = interior width); the reference's SparseLU is
// replaced by LAPACK's banded LU with partial pivoting (dgbsv).
SchurData leaf_schur(const GridBox& box, const Operator& op) {
  SchurData out;
  out.box_id = box.id;
  out.x0 = box.x0; out.x1 = box.x1; out.y0 = box.y0; out.y1 = box.y1;
  out.boundary = box.boundary;
  const Index nb = Index(box.boundary.size()), ni = Index(box.interior.size());
  Mat abb(nb, nb);
  for (Index i = 0; i < nb; ++i)
    for (Index j = 0; j < nb; ++j) abb(i, j) = op.coeff(box.boundary[i], box.boundary[j]);
  if (ni == 0) { out.S = std::move(abb); return out; }
  std::unordered_map<Index, Index> ipos, bpos;
  for (Index i = 0; i < ni; ++i) ipos[box.interior[i]] = i;
  for (Index i = 0; i < nb; ++i) bpos[box.boundary[i]] = i;
  const int64_t w = box.x1 - box.x0 - 1;  // interior width = half bandwidth
  const int64_t kl = w, ku = w, ldab = 2 * kl + ku + 1;
  std::vector<double> ab(size_t(ldab) * ni, 0.0);
  Mat aib(ni, nb), abi(nb, ni);
  for (Index i = 0; i < ni; ++i) {
    const Index row = box.interior[i];
    const GridPoint p = op.lat.point_of(row);
    const std::array<GridPoint, 5> cols{GridPoint{p.x, p.y}, GridPoint{p.x + 1, p.y}, GridPoint{p.x - 1, p.y},
                                        GridPoint{p.x, p.y + 1}, GridPoint{p.x, p.y - 1}};
    for (const auto& q : cols) {
      if (!op.lat.is_unknown(q.x, q.y)) continue;
      const Index col = op.lat.unknown_id(q.x, q.y);
      const double v = op.coeff(row, col);
      if (auto it = ipos.find(col); it != ipos.end()) {
        const Index j = it->second;
        ab[size_t(j) * ldab + (kl + ku + i - j)] = v;  // LAPACK band storage
      } else if (auto bb = bpos.find(col); bb != bpos.end()) {
        aib(i, bb->second) = v;
        abi(bb->second, i) = op.coeff(col, row);
      }  // couplings leaving the box belong to later merges (dense_nd.cpp:85)
    }
  }
  std::vector<int64_t> ipiv(ni);
  int64_t info = 0, n64 = ni, nrhs = nb;
  Mat x = aib;
  scipy_dgbsv_64_(&n64, &kl, &ku, &nrhs, ab.data(), &ldab, ipiv.data(), x.a.data(), &n64, &info);
  if (info != 0) throw FactorizationError("interior block A_ii is singular", "leaf box " + std::to_string(box.id));
  gemm_sub(abi, x, abb);
  out.S = std::move(abb);
  return out;
}

std::string box_label(int level, int box) { return "level " + std::to_string(level) + " box " + std::to_string(box); }

// merge_two (dense_nd.cpp:105-186)
SchurData merge_two(const SchurData& a, const SchurData& b, const Operator& op, int level, int box) {
  const Lattice lat = op.lat;
  SchurData out;
  out.x0 = std::min(a.x0, b.x0); out.x1 = std::max(a.x1, b.x1);
  out.y0 = std::min(a.y0, b.y0); out.y1 = std::max(a.y1, b.y1);
  std::unordered_map<Index, Index> pos;
  std::vector<Index> nodes;
  for (const auto& gp : rect_perimeter_ccw(out.x0, out.x1, out.y0, out.y1)) {
    const Index id = lat.unknown_id(gp.x, gp.y);
    pos[id] = Index(nodes.size());
    nodes.push_back(id);
    out.boundary.push_back(id);
  }
  const Index nb = Index(out.boundary.size());
  for (const auto* child : {&a, &b})
    for (Index id : child->boundary)
      if (!pos.count(id)) { pos[id] = Index(nodes.size()); nodes.push_back(id); }
  const Index total = Index(nodes.size()), ni = total - nb;
  Mat m(total, total);
  for (const auto* child : {&a, &b}) {
    const Index cn = Index(child->boundary.size());
    std::vector<Index> p(cn);
    for (Index i = 0; i < cn; ++i) p[i] = pos.at(child->boundary[i]);
    for (Index j = 0; j < cn; ++j)
      for (Index i = 0; i < cn; ++i) m(p[i], p[j]) += child->S(i, j);
  }
  std::unordered_map<Index, char> in_a;  // cross couplings (dense_nd.cpp:148-165)
  for (Index id : a.boundary) in_a[id] = 1;
  for (Index id : b.boundary) {
    const GridPoint gp = lat.point_of(id);
    const std::array<GridPoint, 4> nbs{GridPoint{gp.x + 1, gp.y}, GridPoint{gp.x - 1, gp.y},
                                       GridPoint{gp.x, gp.y + 1}, GridPoint{gp.x, gp.y - 1}};
    for (const auto& q : nbs) {
      if (!lat.is_unknown(q.x, q.y)) continue;
      const Index qid = lat.unknown_id(q.x, q.y);
      if (!in_a.count(qid)) continue;
      m(pos.at(id), pos.at(qid)) += op.coeff(id, qid);
      m(pos.at(qid), pos.at(id)) += op.coeff(qid, id);
    }
  }
  Mat mbb(nb, nb), mbi(nb, ni), mib(ni, nb), mii(ni, ni);
  for (Index j = 0; j < total; ++j)
    for (Index i = 0; i < total; ++i) {
      const double v = m(i, j);
      if (i < nb && j < nb) mbb(i, j) = v;
      else if (i < nb) mbi(i, j - nb) = v;
      else if (j < nb) mib(i - nb, j) = v;
      else mii(i - nb, j - nb) = v;
    }
  if (ni == 0) { out.S = std::move(mbb); return out; }
  std::vector<int64_t> ipiv(ni);
  int64_t n64 = ni, info = 0, nrhs = nb;
  scipy_dgetrf_64_(&n64, &n64, mii.a.data(), &n64, ipiv.data(), &info);
  double pmin = INFINITY, pmax = 0.0;
  for (Index i = 0; i < ni; ++i) {
    const double d = std::abs(mii(i, i));
    pmin = std::min(pmin, d);
    pmax = std::max(pmax, d);
  }
  if (!(pmin > pmax * 1e-300) || !std::isfinite(pmax))  // dense_nd.cpp:175-180
    throw FactorizationError("interface block is singular", box_label(level, box));
  static const bool left_assoc = std::getenv("ORC_RIGHT_LOOKING_ASSOC") != nullptr;
  if (!left_assoc) {  // reference association: S = M_bb - M_bi (U^-1 L^-1 P M_ib)
    scipy_dgetrs_64_("N", &n64, &nrhs, mii.a.data(), &n64, ipiv.data(), mib.a.data(), &n64, &info, 1);
    gemm_sub(mbi, mib, mbb);
  } else {  // diagnostic: S = M_bb - (M_bi U^-1)(L^-1 P M_ib), the right-looking association
    const int64_t one = 1, nb64 = nb;
    const double alpha = 1.0;
    scipy_dlaswp_64_(&nrhs, mib.a.data(), &n64, &one, &n64, ipiv.data(), &one);
    scipy_dtrsm_64_("L", "L", "N", "U", &n64, &nrhs, &alpha, mii.a.data(), &n64, mib.a.data(), &n64, 1, 1, 1, 1);
    scipy_dtrsm_64_("R", "U", "N", "N", &nb64, &n64, &alpha, mii.a.data(), &n64, mbi.a.data(), &nb64, 1, 1, 1, 1);
    gemm_sub(mbi, mib, mbb);
  }
  out.S = std::move(mbb);
  return out;
}

// Bounded pool: one level's boxes spread over `threads` workers (the
// reference's accel engine does the same, accel_nd.cpp:635-659).
void parallel_for(int count, int threads, const std::function<void(int)>& fn) {
  if (threads <= 1 || count <= 1) { for (int i = 0; i < count; ++i) fn(i); return; }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(threads);
  std::atomic<int> next{0};
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int i = next++; i < count; i = next++) fn(i);
      } catch (...) { errs[t] = std::current_exception(); }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs) if (e) std::rethrow_exception(e);
}

struct Result {
  SchurData root;
  Mat G;
  double cond = 0.0;
  std::unordered_map<int, SchurData> all;  // every box (keep_all)
  double seconds_build = 0.0, seconds_inverse = 0.0;
};

// build_root_dense (dense_nd.cpp:196-225). mode 0: boxes serial, BLAS on
// `threads` cores (best-effort host); mode 1: boxes of a level spread over
// `threads` workers with 1 BLAS thread each (the reference's own threading);
// mode 2 (best CPU baseline): mode 1 on levels with >= threads boxes, mode 0
// on the few-box top levels.
Result build_root_dense(const Operator& op, const BoxTree& tree, int threads, int mode, bool keep_all) {
  const auto t0 = std::chrono::steady_clock::now();
  int box_threads = mode == 1 ? threads : 1;
  auto set_level_mode = [&](size_t boxes) {
    const bool by_box = mode == 1 || (mode == 2 && boxes >= size_t(threads));
    box_threads = by_box ? threads : 1;
    scipy_openblas_set_num_threads64_(by_box ? 1 : threads);
  };
  set_level_mode(tree.levels[tree.depth].size());
  Result res;
  std::vector<SchurData> current(tree.levels[tree.depth].size());
  parallel_for(int(current.size()), box_threads, [&](int i) {
    current[i] = leaf_schur(tree.boxes[tree.levels[tree.depth][i]], op);
  });
  if (keep_all) for (auto& s : current) res.all[s.box_id] = s;
  for (int lev = tree.depth - 1; lev >= 0; --lev) {
    std::unordered_map<int, const SchurData*> by_box;
    for (const auto& s : current) by_box[s.box_id] = &s;
    std::vector<SchurData> next(tree.levels[lev].size());
    set_level_mode(next.size());
    parallel_for(int(next.size()), box_threads, [&](int i) {
      const int id = tree.levels[lev][i];
      const auto& box = tree.boxes[id];
      const SchurData& sw = *by_box.at(box.children[0]);
      const SchurData& se = *by_box.at(box.children[1]);
      const SchurData& nw = *by_box.at(box.children[2]);
      const SchurData& ne = *by_box.at(box.children[3]);
      const SchurData west = merge_two(sw, nw, op, lev, id);  // merge_four, dense_nd.cpp:188-194
      const SchurData east = merge_two(se, ne, op, lev, id);
      SchurData merged = merge_two(west, east, op, lev, id);
      merged.box_id = id;
      next[i] = std::move(merged);
    });
    current = std::move(next);
    if (keep_all) for (auto& s : current) res.all[s.box_id] = s;
  }
  scipy_openblas_set_num_threads64_(threads);
  const auto t1 = std::chrono::steady_clock::now();
  res.root = std::move(current.front());
  const Index nb = Index(res.root.boundary.size());
  Mat lu = res.root.S;
  res.G = Mat(nb, nb);
  for (Index i = 0; i < nb; ++i) res.G(i, i) = 1.0;
  std::vector<int64_t> ipiv(nb);
  int64_t n64 = nb, info = 0;
  if (nb > 0) {
    scipy_dgetrf_64_(&n64, &n64, lu.a.data(), &n64, ipiv.data(), &info);
    scipy_dgetrs_64_("N", &n64, &n64, lu.a.data(), &n64, ipiv.data(), res.G.a.data(), &n64, &info, 1);
  }
  auto norm1 = [&](const Mat& x) {
    double best = 0.0;
    for (Index j = 0; j < x.cols; ++j) {
      double s = 0.0;
      for (Index i = 0; i < x.rows; ++i) s += std::abs(x(i, j));
      best = std::max(best, s);
    }
    return best;
  };
  res.cond = norm1(res.root.S) * norm1(res.G);  // dense_nd.cpp:222-223
  const auto t2 = std::chrono::steady_clock::now();
  res.seconds_build = std::chrono::duration<double>(t1 - t0).count();
  res.seconds_inverse = std::chrono::duration<double>(t2 - t1).count();
  return res;
}

}  // namespace orc

// ------------------------------------------------------------------ C API
namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const orc::FactorizationError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}
}  // namespace

extern "C" {
const char* orc_last_error() { return g_err.c_str(); }

int orc_problem_create(const char* name, int n, double param, uint64_t seed, void** out) {
  return guarded([&] { *out = new orc::Operator(orc::make_problem(name, n, param, seed)); });
}
void orc_problem_free(void* p) { delete static_cast<orc::Operator*>(p); }
// stencil export: 5 x nu, rows center, east, west, north, south (unknown_id order)
void orc_problem_stencil(void* p, double* out) {
  auto* op = static_cast<orc::Operator*>(p);
  const size_t nu = op->center.size();
  const std::vector<double>* v[5] = {&op->center, &op->east, &op->west, &op->north, &op->south};
  for (int r = 0; r < 5; ++r) std::memcpy(out + r * nu, v[r]->data(), nu * sizeof(double));
}
double orc_problem_coeff(void* p, int64_t row, int64_t col) { return static_cast<orc::Operator*>(p)->coeff(row, col); }

int orc_tree_create(int n, int n_leaf, int uniform_side, void** out) {
  return guarded([&] { *out = new orc::BoxTree(orc::build_tree(n, n_leaf, uniform_side)); });
}
void orc_tree_free(void* t) { delete static_cast<orc::BoxTree*>(t); }
int orc_tree_depth(void* t) { return static_cast<orc::BoxTree*>(t)->depth; }
int orc_tree_num_boxes(void* t) { return int(static_cast<orc::BoxTree*>(t)->boxes.size()); }
int orc_tree_level_size(void* t, int lev) { return int(static_cast<orc::BoxTree*>(t)->levels[lev].size()); }
void orc_tree_level(void* t, int lev, int* ids) {
  const auto& l = static_cast<orc::BoxTree*>(t)->levels[lev];
  std::copy(l.begin(), l.end(), ids);
}
// info: level, parent, c0..c3, x0, x1, y0, y1, gx0, gx1, gy0, gy1, nb, ni
void orc_tree_box(void* t, int id, int64_t* info) {
  const auto& b = static_cast<orc::BoxTree*>(t)->boxes[id];
  const int64_t v[16] = {b.level, b.parent, b.children[0], b.children[1], b.children[2], b.children[3],
                         b.x0, b.x1, b.y0, b.y1, b.gx0, b.gx1, b.gy0, b.gy1,
                         int64_t(b.boundary.size()), int64_t(b.interior.size())};
  std::copy(v, v + 16, info);
}
void orc_tree_box_sets(void* t, int id, int64_t* boundary, int64_t* interior) {
  const auto& b = static_cast<orc::BoxTree*>(t)->boxes[id];
  std::copy(b.boundary.begin(), b.boundary.end(), boundary);
  std::copy(b.interior.begin(), b.interior.end(), interior);
}

int orc_build_dense(void* p, void* t, int threads, int mode, int keep_all, void** out) {
  return guarded([&] {
    *out = new orc::Result(orc::build_root_dense(*static_cast<orc::Operator*>(p), *static_cast<orc::BoxTree*>(t),
                                                 threads, mode, keep_all != 0));
  });
}
void orc_result_free(void* r) { delete static_cast<orc::Result*>(r); }
int64_t orc_result_nb(void* r) { return int64_t(static_cast<orc::Result*>(r)->root.boundary.size()); }
void orc_result_root(void* r, int64_t* boundary, double* S, double* G, double* cond, double* secs) {
  auto* res = static_cast<orc::Result*>(r);
  std::copy(res->root.boundary.begin(), res->root.boundary.end(), boundary);
  if (S) std::copy(res->root.S.a.begin(), res->root.S.a.end(), S);
  if (G) std::copy(res->G.a.begin(), res->G.a.end(), G);
  *cond = res->cond;
  secs[0] = res->seconds_build;
  secs[1] = res->seconds_inverse;
}
// S of any box kept with keep_all (column-major nb x nb); returns nb or -1
int64_t orc_result_box(void* r, int box_id, double* S) {
  auto* res = static_cast<orc::Result*>(r);
  auto it = res->all.find(box_id);
  if (it == res->all.end()) return -1;
  if (S) std::copy(it->second.S.a.begin(), it->second.S.a.end(), S);
  return int64_t(it->second.boundary.size());
}

// Single-box helpers for the reference's unit tests (test_dense_nd.cpp):
// leaf_schur on an arbitrary rectangle, and merge_two of two rectangles
// (each eliminated from scratch as a leaf first).
int orc_leaf_rect(void* p, int x0, int x1, int y0, int y1, double* S, int64_t* nb_out) {
  return guarded([&] {
    auto* op = static_cast<orc::Operator*>(p);
    orc::GridBox box;
    box.id = 0;
    box.x0 = x0; box.x1 = x1; box.y0 = y0; box.y1 = y1;
    for (const auto& gp : orc::rect_perimeter_ccw(x0, x1, y0, y1)) box.boundary.push_back(op->lat.unknown_id(gp.x, gp.y));
    for (int y = y0 + 1; y <= y1 - 1; ++y)
      for (int x = x0 + 1; x <= x1 - 1; ++x) box.interior.push_back(op->lat.unknown_id(x, y));
    const auto s = orc::leaf_schur(box, *op);
    *nb_out = int64_t(s.boundary.size());
    if (S) std::copy(s.S.a.begin(), s.S.a.end(), S);
  });
}
int orc_merge_rects(void* p, const int* ra, const int* rb, double* S, int64_t* nb_out) {
  return guarded([&] {
    auto* op = static_cast<orc::Operator*>(p);
    orc::SchurData ch[2];
    const int* rr[2] = {ra, rb};
    for (int c = 0; c < 2; ++c) {
      orc::GridBox box;
      box.x0 = rr[c][0]; box.x1 = rr[c][1]; box.y0 = rr[c][2]; box.y1 = rr[c][3];
      for (const auto& gp : orc::rect_perimeter_ccw(box.x0, box.x1, box.y0, box.y1))
        box.boundary.push_back(op->lat.unknown_id(gp.x, gp.y));
      for (int y = box.y0 + 1; y <= box.y1 - 1; ++y)
        for (int x = box.x0 + 1; x <= box.x1 - 1; ++x) box.interior.push_back(op->lat.unknown_id(x, y));
      ch[c] = orc::leaf_schur(box, *op);
    }
    const auto s = orc::merge_two(ch[0], ch[1], *op, -1, -1);
    *nb_out = int64_t(s.boundary.size());
    if (S) std::copy(s.S.a.begin(), s.S.a.end(), S);
  });
}
// merge_two of two given Schur complements on rectangles ra, rb (x0,x1,y0,y1)
// (column-major, CCW boundary order) — the top-of-tree merges of a sharded build.
int orc_merge_given(void* p, const int* ra, const double* Sa, const int* rb, const double* Sb, double* S,
                    int64_t* nb_out) {
  return guarded([&] {
    auto* op = static_cast<orc::Operator*>(p);
    orc::SchurData ch[2];
    const int* rr[2] = {ra, rb};
    const double* ss[2] = {Sa, Sb};
    for (int c = 0; c < 2; ++c) {
      ch[c].x0 = rr[c][0]; ch[c].x1 = rr[c][1]; ch[c].y0 = rr[c][2]; ch[c].y1 = rr[c][3];
      for (const auto& gp : orc::rect_perimeter_ccw(ch[c].x0, ch[c].x1, ch[c].y0, ch[c].y1))
        ch[c].boundary.push_back(op->lat.unknown_id(gp.x, gp.y));
      const int64_t nb = int64_t(ch[c].boundary.size());
      ch[c].S = orc::Mat(nb, nb);
      std::copy(ss[c], ss[c] + nb * nb, ch[c].S.a.begin());
    }
    const auto out = orc::merge_two(ch[0], ch[1], *op, -1, -1);
    *nb_out = int64_t(out.boundary.size());
    if (S) std::copy(out.S.a.begin(), out.S.a.end(), S);
  });
}
int orc_blas_threads() { return scipy_openblas_get_num_threads64_(); }

// Probe vectors of error_metrics (reference.cpp:139-161): seeded random unit
// boundary vector (mt19937_64, Box-Muller on explicit uniforms) and the smooth one.
void orc_random_unit_boundary(int64_t size, uint64_t seed, double* r) {
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
  for (int64_t i = 0; i < size; i += 2) {
    const double u1 = (double(rng() >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = double(rng() >> 11) * 0x1.0p-53;
    const double rad = std::sqrt(-2.0 * std::log(u1));
    r[i] = rad * std::cos(2.0 * std::numbers::pi * u2);
    if (i + 1 < size) r[i + 1] = rad * std::sin(2.0 * std::numbers::pi * u2);
  }
  double nrm = 0.0;
  for (int64_t i = 0; i < size; ++i) nrm += r[i] * r[i];
  nrm = std::sqrt(nrm);
  for (int64_t i = 0; i < size; ++i) r[i] /= nrm;
}
void orc_smooth_boundary(int64_t size, double* r) {
  double nrm = 0.0;
  for (int64_t i = 0; i < size; ++i) {
    r[i] = std::sin(2.0 * std::numbers::pi * double(i) / double(size));
    nrm += r[i] * r[i];
  }
  nrm = std::sqrt(nrm);
  for (int64_t i = 0; i < size; ++i) r[i] /= nrm;
}
}
