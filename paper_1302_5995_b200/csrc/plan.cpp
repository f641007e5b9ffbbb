// Build plan (see plan.hpp). Geometry follows the reference:
//   unknown ids        grid.hpp:68-70   (y-1)(n-2) + (x-1)
//   CCW perimeter      grid.cpp:170-190
//   quadtree           grid.cpp:213-266 (halve the full grid, left/south take the extra point)
//   box index sets     grid.cpp:194-209
//   merge ordering     dense_nd.cpp:114-131 (union boundary CCW, then the remaining
//                      child boundary nodes, child a first)
//   merge_four order   dense_nd.cpp:188-194 (SW+NW, SE+NE, W|E)
#include <cstdlib>
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>

namespace dtnb {

// DTN_SKETCH_SPLIT=0: the structured boxes' sketches as one K = nb product per box
static bool sketch_split_off() {
  static const bool off = [] {
    const char* e = std::getenv("DTN_SKETCH_SPLIT");
    return e && std::atoi(e) == 0;
  }();
  return off;
}


void perimeter_ccw(const Rect& r, std::vector<std::pair<int, int>>& p) {
  p.clear();
  if (r.empty()) return;
  if (r.x0 == r.x1 && r.y0 == r.y1) { p.push_back({r.x0, r.y0}); return; }
  if (r.x0 == r.x1) { for (int y = r.y0; y <= r.y1; ++y) p.push_back({r.x0, y}); return; }
  if (r.y0 == r.y1) { for (int x = r.x0; x <= r.x1; ++x) p.push_back({x, r.y0}); return; }
  for (int x = r.x0; x <= r.x1; ++x) p.push_back({x, r.y0});
  for (int y = r.y0 + 1; y <= r.y1; ++y) p.push_back({r.x1, y});
  for (int x = r.x1 - 1; x >= r.x0; --x) p.push_back({x, r.y1});
  for (int y = r.y1 - 1; y >= r.y0 + 1; --y) p.push_back({r.x0, y});
}

int perimeter_size(const Rect& r) {
  if (r.empty()) return 0;
  if (r.w() == 1 || r.h() == 1) return int(r.nodes());
  return 2 * (r.w() + r.h()) - 4;
}

namespace {

// Closed-form position of (x,y) in perimeter_ccw(r); (x,y) must lie on it.
int ccw_index(const Rect& r, int x, int y) {
  const int w = r.w(), h = r.h();
  if (w == 1) return y - r.y0;
  if (h == 1) return x - r.x0;
  if (y == r.y0) return x - r.x0;
  if (x == r.x1) return (w - 1) + (y - r.y0);
  if (y == r.y1) return (w - 1) + (h - 1) + (r.x1 - x);
  return 2 * (w - 1) + (h - 1) + (r.y1 - y);
}

bool on_perimeter(const Rect& r, int x, int y) { return x == r.x0 || x == r.x1 || y == r.y0 || y == r.y1; }

struct Builder {
  const PlanKey& key;
  Plan& P;
  int side;  // n - 2
  std::vector<std::pair<int, int>> tmp;

  Builder(const PlanKey& k, Plan& p) : key(k), P(p), side(k.n - 2) {}

  int32_t gid(int x, int y) const { return int32_t(int64_t(y - 1) * side + (x - 1)); }

  int add_micro(const Rect& r, int leaf_box) {
    Node nd;
    nd.kind = NodeKind::micro;
    nd.r = r;
    nd.nb = perimeter_size(r);
    nd.total = int(r.nodes());
    nd.ni = nd.total - nd.nb;
    nd.ref_box = -1;
    nd.label_box = leaf_box;
    nd.pos_off = int64_t(P.pos.size());
    for (int y = r.y0 + 1; y <= r.y1 - 1; ++y)
      for (int x = r.x0 + 1; x <= r.x1 - 1; ++x) P.pos.push_back({0, -1, gid(x, y), 0});
    perimeter_ccw(r, tmp);
    for (auto [x, y] : tmp) P.pos.push_back({0, -1, gid(x, y), 0});
    P.micro_flops += merge_flop_count(nd.ni, nd.nb);
    P.nodes.push_back(nd);
    return int(P.nodes.size()) - 1;
  }

  // merge_two (dense_nd.cpp:105-186) as a DAG node
  int add_merge(int ia, int ib, int label_level, int label_box, bool tree_merge) {
    if (ia < 0) return ib;
    if (ib < 0) return ia;
    const Rect ra = P.nodes[ia].r, rb = P.nodes[ib].r;
    Rect u{std::min(ra.x0, rb.x0), std::max(ra.x1, rb.x1), std::min(ra.y0, rb.y0), std::max(ra.y1, rb.y1)};
    if (u.nodes() != ra.nodes() + rb.nodes())
      throw std::invalid_argument("merge_two: children do not tile a rectangle");
    Node nd;
    nd.kind = NodeKind::merge;
    nd.r = u;
    nd.a = ia;
    nd.b = ib;
    nd.nb = perimeter_size(u);
    const int na = P.nodes[ia].nb, nbb = P.nodes[ib].nb;
    nd.total = na + nbb;
    nd.ni = nd.total - nd.nb;
    nd.label_level = label_level;
    nd.label_box = label_box;
    nd.ref_box = -1;
    nd.pos_off = int64_t(P.pos.size());
    P.pos.resize(P.pos.size() + nd.total, PosEntry{0, -1, 0, 0});
    PosEntry* pe = P.pos.data() + nd.pos_off;
    std::vector<int> posA(na), posB(nbb);
    int next_int = 0;
    for (int c = 0; c < 2; ++c) {
      const Rect& rc = c == 0 ? ra : rb;
      std::vector<int>& pm = c == 0 ? posA : posB;
      perimeter_ccw(rc, tmp);
      for (int i = 0; i < int(tmp.size()); ++i) {
        const auto [x, y] = tmp[i];
        const int p = on_perimeter(u, x, y) ? nd.ni + ccw_index(u, x, y) : next_int++;
        pm[i] = p;
        pe[p].src = c == 0 ? i : -i - 1;
        pe[p].gid = gid(x, y);
      }
    }
    if (next_int != nd.ni) throw std::logic_error("merge_two: interface bookkeeping");
    // couplings across the shared edge (dense_nd.cpp:148-165); exactly one
    // partner per interface node for the 5-point stencil
    auto couple = [&](int xa, int ya, int xb, int yb, int dir_ab, int dir_ba) {
      const int pa = posA[ccw_index(ra, xa, ya)], pb = posB[ccw_index(rb, xb, yb)];
      pe[pa].partner = pb;
      pe[pa].dir = dir_ab;
      pe[pb].partner = pa;
      pe[pb].dir = dir_ba;
    };
    if (ra.x1 + 1 == rb.x0 && ra.y0 == rb.y0 && ra.y1 == rb.y1) {
      for (int y = ra.y0; y <= ra.y1; ++y) couple(ra.x1, y, rb.x0, y, 1, 2);
    } else if (rb.x1 + 1 == ra.x0 && ra.y0 == rb.y0 && ra.y1 == rb.y1) {
      for (int y = ra.y0; y <= ra.y1; ++y) couple(ra.x0, y, rb.x1, y, 2, 1);
    } else if (ra.y1 + 1 == rb.y0 && ra.x0 == rb.x0 && ra.x1 == rb.x1) {
      for (int x = ra.x0; x <= ra.x1; ++x) couple(x, ra.y1, x, rb.y0, 3, 4);
    } else if (rb.y1 + 1 == ra.y0 && ra.x0 == rb.x0 && ra.x1 == rb.x1) {
      for (int x = ra.x0; x <= ra.x1; ++x) couple(x, ra.y0, x, rb.y1, 4, 3);
    } else {
      throw std::invalid_argument("merge_two: children are not edge-adjacent");
    }
    nd.wave = 1 + std::max(P.nodes[ia].wave, P.nodes[ib].wave);
    if (tree_merge) P.merge_flops += merge_flop_count(nd.ni, nd.nb);
    else P.micro_flops += merge_flop_count(nd.ni, nd.nb);
    P.nodes.push_back(nd);
    return int(P.nodes.size()) - 1;
  }

  // Leaf elimination below a reference leaf: binary splits of the longer
  // side until a box fits one CTA (micro_max unknowns).
  int leaf_node(const Rect& r, int leaf_box) {
    if (r.empty()) return -1;
    if (r.nodes() <= key.micro_max) return add_micro(r, leaf_box);
    Rect lo = r, hi = r;
    if (r.w() >= r.h()) {
      const int wl = r.w() / 2;
      lo.x1 = r.x0 + wl - 1;
      hi.x0 = r.x0 + wl;
    } else {
      const int hl = r.h() / 2;
      lo.y1 = r.y0 + hl - 1;
      hi.y0 = r.y0 + hl;
    }
    const int a = leaf_node(lo, leaf_box), b = leaf_node(hi, leaf_box);
    return add_merge(a, b, -1, leaf_box, false);
  }
};

void build_ref_tree(const PlanKey& key, Plan& P) {
  const int n = key.n;
  if (n < 4) throw std::invalid_argument("build_tree: n must be >= 4");
  int depth = 0;
  const bool uniform = key.leaf_side > 0;
  if (uniform) {
    int s = n - 2;
    while (s > key.leaf_side) {
      if (s % 2) throw std::invalid_argument("build_tree: n-2 is not leaf_side * 2^L");
      s /= 2;
      ++depth;
    }
    if (s != key.leaf_side) throw std::invalid_argument("build_tree: n-2 is not leaf_side * 2^L");
  } else {
    if (key.n_leaf < 16) throw std::invalid_argument("build_tree: n_leaf must be >= 16");
    while (double(n) * n > double(key.n_leaf) * std::pow(4.0, depth)) ++depth;  // grid.cpp:217-218
  }
  P.depth = depth;
  P.levels.assign(depth + 1, {});
  auto fill = [&](RefBox& b) {  // grid.cpp:194-209
    b.r.x0 = std::max(b.gx0, 1);
    b.r.y0 = std::max(b.gy0, 1);
    b.r.x1 = std::min(b.gx1, n - 1) - 1;
    b.r.y1 = std::min(b.gy1, n - 1) - 1;
  };
  RefBox root;
  root.id = 0;
  root.gx0 = uniform ? 1 : 0;
  root.gx1 = uniform ? n - 1 : n;
  root.gy0 = root.gx0;
  root.gy1 = root.gx1;
  fill(root);
  P.boxes.push_back(root);
  P.levels[0].push_back(0);
  for (int lev = 0; lev < depth; ++lev) {
    for (int id : P.levels[lev]) {
      const RefBox pb = P.boxes[id];
      const int xm = uniform ? pb.gx0 + (pb.gx1 - pb.gx0) / 2 : pb.gx0 + (pb.gx1 - pb.gx0 + 1) / 2;
      const int ym = uniform ? pb.gy0 + (pb.gy1 - pb.gy0) / 2 : pb.gy0 + (pb.gy1 - pb.gy0 + 1) / 2;
      const int reg[4][4] = {{pb.gx0, xm, pb.gy0, ym}, {xm, pb.gx1, pb.gy0, ym},
                             {pb.gx0, xm, ym, pb.gy1}, {xm, pb.gx1, ym, pb.gy1}};
      for (int c = 0; c < 4; ++c) {
        RefBox ch;
        ch.id = int(P.boxes.size());
        ch.level = lev + 1;
        ch.parent = id;
        ch.gx0 = reg[c][0]; ch.gx1 = reg[c][1]; ch.gy0 = reg[c][2]; ch.gy1 = reg[c][3];
        fill(ch);
        P.boxes[id].children[c] = ch.id;
        P.levels[lev + 1].push_back(ch.id);
        P.boxes.push_back(ch);
      }
    }
  }
}

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace

void root_halves(const PlanKey& key, int* depth, int* nb_w, int* nb_e) {
  Plan P;
  build_ref_tree(key, P);
  *depth = P.depth;
  *nb_w = *nb_e = 0;
  if (P.depth == 0) return;
  const RefBox& rt = P.boxes[0];
  const Rect& sw = P.boxes[rt.children[0]].r;
  const Rect& se = P.boxes[rt.children[1]].r;
  const Rect& nw = P.boxes[rt.children[2]].r;
  const Rect& ne = P.boxes[rt.children[3]].r;
  auto uni = [](const Rect& a, const Rect& b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    return Rect{std::min(a.x0, b.x0), std::max(a.x1, b.x1), std::min(a.y0, b.y0), std::max(a.y1, b.y1)};
  };
  *nb_w = perimeter_size(uni(sw, nw));
  *nb_e = perimeter_size(uni(se, ne));
}

std::vector<int> shard_nodes(const Plan& P, int nshards) {
  auto need = [&](bool ok) {
    if (!ok) throw std::invalid_argument("shards: the tree is too shallow for this shard count");
  };
  const Node& root = P.nodes[P.root];
  switch (nshards) {
    case 1:
      return {P.root};
    case 2:  // W | E halves of the root's merge_four (dense_nd.cpp:188-194)
      need(root.kind == NodeKind::merge && P.depth >= 1);
      return {root.a, root.b};
    case 4: {  // quadrants SW, SE, NW, NE
      need(P.depth >= 1);
      std::vector<int> out;
      for (int c = 0; c < 4; ++c) out.push_back(P.boxes[P.boxes[0].children[c]].node);
      return out;
    }
    case 8: {  // W | E halves of every quadrant
      need(P.depth >= 2);
      std::vector<int> out;
      for (int c = 0; c < 4; ++c) {
        const Node& q = P.nodes[P.boxes[P.boxes[0].children[c]].node];
        need(q.kind == NodeKind::merge);
        out.push_back(q.a);
        out.push_back(q.b);
      }
      return out;
    }
    default:
      throw std::invalid_argument("shards: nshards must be 1, 2, 4 or 8");
  }
}

Plan make_plan(const PlanKey& key) {
  if (key.nloads < 0 || key.micro_max + key.nloads > key.small_max)
    throw std::invalid_argument("build: too many body loads for the fused leaf kernel (micro_max + loads > " +
                                std::to_string(key.small_max) + ")");
  if (key.micro_max < 4 || key.micro_max > key.small_max)
    throw std::invalid_argument("make_plan: bad micro/small thresholds");
  Plan P;
  P.key = key;
  P.n = key.n;
  build_ref_tree(key, P);
  Builder B(key, P);
  // bottom-up over the reference tree (build_root_dense, dense_nd.cpp:196-216)
  for (int lev = P.depth; lev >= 0; --lev) {
    for (int id : P.levels[lev]) {
      RefBox& bx = P.boxes[id];
      const int before = int(P.nodes.size());
      if (lev == P.depth) {
        bx.node = B.leaf_node(bx.r, id);
      } else {
        const int sw = P.boxes[bx.children[0]].node, se = P.boxes[bx.children[1]].node;
        const int nw = P.boxes[bx.children[2]].node, ne = P.boxes[bx.children[3]].node;
        const int w = B.add_merge(sw, nw, lev, id, true);
        const int e = B.add_merge(se, ne, lev, id, true);
        // merge_four's halves merge W|E next: their J edges face each other
        // (build_root_accel's merge_pair(..., JSide::east / west), accel_nd.cpp:771-776)
        if (w >= before) P.nodes[w].jside = 2;
        if (e >= before) P.nodes[e].jside = 3;
        bx.node = B.add_merge(w, e, lev, id, true);
      }
      // a box's own J edge faces its sibling in the next merge_four: SW / SE merge
      // upward (north), NW / NE downward (child_j_side, accel_nd.cpp:661-665)
      if (bx.node >= before && lev > 0) {
        const RefBox& par = P.boxes[bx.parent];
        const int ci = int(std::find(par.children, par.children + 4, id) - par.children);
        P.nodes[bx.node].jside = ci < 2 ? 0 : 1;
      }
      if (bx.node >= 0 && P.nodes[bx.node].ref_box < 0) P.nodes[bx.node].ref_box = id;
    }
  }
  P.root = P.boxes[0].node;
  if (P.root < 0) throw std::invalid_argument("make_plan: empty domain");
  P.active.assign(P.nodes.size(), 1);
  if (key.nshards > 1 || key.shard >= 0) {
    const std::vector<int> sh = shard_nodes(P, key.nshards);
    std::vector<char> below(P.nodes.size(), 0);  // inside some shard's subtree (inclusive)
    std::vector<int> stack;
    for (int s0 : sh) {
      stack.push_back(s0);
      while (!stack.empty()) {
        const int v = stack.back();
        stack.pop_back();
        if (v < 0 || below[v]) continue;
        below[v] = 1;
        if (P.nodes[v].kind == NodeKind::merge) {
          stack.push_back(P.nodes[v].a);
          stack.push_back(P.nodes[v].b);
        }
      }
    }
    if (key.shard >= 0) {
      if (key.shard >= int(sh.size())) throw std::invalid_argument("shards: shard index out of range");
      std::vector<char> mine(P.nodes.size(), 0);
      stack.push_back(sh[key.shard]);
      while (!stack.empty()) {
        const int v = stack.back();
        stack.pop_back();
        if (v < 0 || mine[v]) continue;
        mine[v] = 1;
        if (P.nodes[v].kind == NodeKind::merge) {
          stack.push_back(P.nodes[v].a);
          stack.push_back(P.nodes[v].b);
        }
      }
      P.active = mine;
      P.root = sh[key.shard];
    } else {
      for (size_t v = 0; v < P.nodes.size(); ++v) P.active[v] = !below[v];
      P.inputs = sh;
    }
    P.merge_flops = P.micro_flops = 0.0;
    for (size_t v = 0; v < P.nodes.size(); ++v) {
      if (!P.active[v]) continue;
      const Node& nd = P.nodes[v];
      (nd.label_level >= 0 ? P.merge_flops : P.micro_flops) += merge_flop_count(nd.ni, nd.nb);
    }
  }
  // parents (the consumer of each node's S)
  for (int i = 0; i < int(P.nodes.size()); ++i) {
    const Node& nd = P.nodes[i];
    if (nd.kind == NodeKind::merge) {
      P.nodes[nd.a].parent = i;
      P.nodes[nd.b].parent = i;
    }
  }
  std::vector<char> is_input(P.nodes.size(), 0);
  for (int v : P.inputs) is_input[v] = 1;
  for (auto& nd : P.nodes) {
    nd.pos_n = nd.kind == NodeKind::merge ? nd.ni + nd.nb : nd.total;
    nd.sys_nb = nd.nb;
  }
  // compressed engine: structured boxes and structured merges, bottom-up in build
  // order (merge_pair, accel_nd.cpp:667-689; leaves :728-744): a merge of two
  // structured boxes is structured (accel_merge); otherwise the merge is dense and its
  // result is compressed (compress_box) when it has a next merge and size >= crossover
  if (key.structured) {
    for (int i = 0; i < int(P.nodes.size()); ++i) {
      Node& nd = P.nodes[i];
      if (!P.active[i] && !is_input[i]) continue;
      const bool tree_box = nd.label_level >= 0 || nd.ref_box >= 0;  // a reference box or a W/E half
      if (!tree_box || is_input[i]) continue;
      const bool kids = nd.kind == NodeKind::merge && P.active[nd.a] && P.active[nd.b] &&
                        (P.nodes[nd.a].factors || P.nodes[nd.a].exact) &&
                        (P.nodes[nd.b].factors || P.nodes[nd.b].exact) && !is_input[nd.a] && !is_input[nd.b];
      // a structured merge needs both children in factored form; children whose factors
      // would be full rank ("exact") merge densely -- the same result, fewer flops
      nd.smerge = kids && P.nodes[nd.a].factors && P.nodes[nd.b].factors;
      if (nd.jside >= 0 && nd.r.w() >= 3 && nd.r.h() >= 3 && (kids || nd.nb >= key.crossover)) {
        nd.factors = true;
        const int w = nd.r.w(), h = nd.r.h();
        switch (nd.jside) {
          case 0: nd.j0 = w + h - 1; nd.jn = w - 2; break;       // north, x1-1 .. x0+1
          case 1: nd.j0 = 1; nd.jn = w - 2; break;               // south, x0+1 .. x1-1
          case 2: nd.j0 = w; nd.jn = h - 2; break;               // east, y0+1 .. y1-1
          default: nd.j0 = 2 * w + h - 2; nd.jn = h - 2; break;  // west, y1-1 .. y0+1
        }
        int ell = key.ell_base;
        for (int t = 256; t <= nd.jn; t *= 2) ell += key.ell_step;
        ell = int(align_up(ell, 8));
        for (const auto& [jn, e] : key.ell_over)
          if (jn == nd.jn) ell = std::max(ell, e);
        nd.ell = std::min({ell, nd.jn, 252});  // (+ 4 probes <= the QR kernel's 256 columns)
        if (2 * nd.ell >= nd.jn) {  // rank >= half the edge: no compression to gain, keep S exact
          nd.factors = false;
          nd.exact = true;
          nd.ell = nd.jn;
        }
      }
    }
    for (auto& nd : P.nodes)
      if (nd.smerge) {
        const Node& a = P.nodes[nd.a];
        const Node& b = P.nodes[nd.b];
        nd.sys_nb = a.ell + b.ell;
        nd.total = nd.ni + nd.sys_nb;
        // the interface rows are J_a then J_b, each in its box's CCW order
        // (interface_coupling's anti-diagonal pairing, accel_nd.cpp:169-215)
        bool ok = a.jn + b.jn == nd.ni;
        for (int i = 0; ok && i < nd.ni; ++i) {
          const int src = P.pos[size_t(nd.pos_off + i)].src;
          ok = i < a.jn ? src == a.j0 + i : src == -(b.j0 + i - a.jn) - 1;
        }
        if (!ok) throw std::logic_error("structured merge: interface is not the children's J edges");
      }
  }
  // waves
  int nw = 0;
  for (auto& nd : P.nodes) nw = std::max(nw, nd.wave + 1);
  P.waves.assign(nw, {});
  const int nl = key.nloads;
  for (int i = 0; i < int(P.nodes.size()); ++i) {
    Node& nd = P.nodes[i];
    if (!P.active[i] || is_input[i]) continue;
    Wave& wv = P.waves[nd.wave];
    if (nd.kind == NodeKind::micro) {
      wv.micro.push_back(i);
    } else if (!nd.smerge && nd.total + nl <= key.small_max) {  // (load columns ride in the same registers)
      wv.small.push_back(i);
    } else {
      nd.blocked = true;
      // collective top build: blocked merges above the shards split their columns
      if (key.world > 1 && !P.inputs.empty() && !nd.smerge) {
        nd.colshard = true;
        nd.cw = (nd.nb + key.world - 1) / key.world;
      }
      wv.blocked.push_back(i);
      if (nd.smerge) wv.smerge.push_back(i);
      wv.max_ni_blocked = std::max(wv.max_ni_blocked, nd.ni);
    }
    if (nd.factors) wv.compress.push_back(i);
  }
  // storage: one arena, packed by liveness -- a node's S (and factors) live from its
  // wave to its parent's wave (children are dropped level by level,
  // dense_nd.cpp:215), scratch only during its own wave; key.keep keeps everything
  struct Arena {
    std::map<int64_t, int64_t> free;  // offset -> size (doubles), coalesced
    int64_t end = 0;
    int64_t get(int64_t n) {
      n = align_up(std::max<int64_t>(n, 1), 32);
      for (auto it = free.begin(); it != free.end(); ++it)
        if (it->second >= n) {
          const int64_t off = it->first, rest = it->second - n;
          free.erase(it);
          if (rest > 0) free[off + n] = rest;
          return off;
        }
      const int64_t off = end;
      end += n;
      return off;
    }
    void put(int64_t off, int64_t n) {
      n = align_up(std::max<int64_t>(n, 1), 32);
      auto it = free.emplace(off, n).first;
      auto nx = std::next(it);
      if (nx != free.end() && it->first + it->second == nx->first) {
        it->second += nx->second;
        free.erase(nx);
      }
      if (it != free.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) {
          pv->second += it->second;
          free.erase(it);
        }
      }
    }
  } arena;
  constexpr int kForever = 1 << 30;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> release(static_cast<size_t>(nw) + 1);
  int64_t sum = 0;
  auto take = [&](int64_t n, int death) {
    const int64_t off = arena.get(n);
    sum += align_up(std::max<int64_t>(n, 1), 32);
    if (death < kForever && !key.keep) release[size_t(std::min(death, nw))].push_back({off, n});
    return off;
  };
  int64_t poff = 0;
  // caller-provided shard S blocks (top mode): compact, resident
  for (int v : P.inputs) {
    Node& nd = P.nodes[v];
    nd.ld = std::max(nd.nb, 1);
    nd.s_off = take(int64_t(nd.ld) * nd.nb, kForever);
  }
  std::vector<std::vector<int>> born(static_cast<size_t>(nw));
  for (int i = 0; i < int(P.nodes.size()); ++i)
    if (P.active[i] && !is_input[i]) born[size_t(P.nodes[i].wave)].push_back(i);
  for (int w = 0; w < nw; ++w) {
    for (auto [off, n] : release[size_t(w)]) arena.put(off, n);  // dead before this wave
    int nfac = 0;  // structured boxes forming factors in this wave (one batched sketch launch)
    for (int i : born[size_t(w)]) nfac += P.nodes[i].factors ? 1 : 0;
    for (int i : born[size_t(w)]) {
      Node& nd = P.nodes[i];
      const bool top = nd.parent < 0 || !P.active[nd.parent] || i == P.root;
      const int death = top ? kForever : P.nodes[nd.parent].wave + 1;  // free after the parent's wave
      if (nd.blocked) {
        if (nd.smerge) {  // reduced interface system (scratch) + the assembled S (kept)
          nd.ldm = int(align_up(nd.total, 8));
          nd.m_off = take(int64_t(nd.ldm) * nd.total, w + 1);
          nd.ld = int(align_up(nd.nb, 8));
          nd.s_off = take(int64_t(nd.ld) * nd.nb, death);
          nd.ldg = int(align_up(nd.nb, 8));
          nd.ldr = int(align_up(nd.sys_nb, 2));
          nd.lkg_off = take(int64_t(nd.ldg) * nd.sys_nb, w + 1);
          nd.rkg_off = take(int64_t(nd.ldr) * nd.nb, w + 1);
          nd.tg_off = take(int64_t(nd.ldg) * nd.sys_nb, w + 1);
          nd.cbuf_off = take(int64_t(nd.ldr) * nd.sys_nb, w + 1);
        } else {
          nd.ldm = int(align_up(nd.total, 8));
          // (column-sharded merges: every rank's chunk is ldm x cw, the gather is in place)
          const int64_t cols = nd.colshard ? std::max<int64_t>(nd.total, nd.ni + int64_t(key.world) * nd.cw)
                                           : nd.total + nl;
          nd.m_off = take(int64_t(nd.ldm) * cols, death);
          nd.s_off = nd.m_off + nd.ni + int64_t(nd.ni) * nd.ldm;
          nd.ld = nd.ldm;
          nd.rhs_off = nd.m_off + nd.ni + int64_t(nd.total) * nd.ldm;
          nd.rhs_ld = nd.ldm;
        }
        nd.piv_off = poff;
        poff += align_up(std::max(nd.ni, 1), 4) + 260;  // ipiv + two per-panel row-move lists + flags
        const int64_t nblk = (nd.ni + 127) / 128;
        nd.uinv_off = take(nblk * 2 * 128 * 128, w + 1);
        nd.t_off = take(int64_t(128) * std::max(nd.sys_nb + nl, 1), w + 1);
      } else {
        nd.ld = std::max(nd.nb, 1);
        nd.s_off = take(int64_t(nd.ld) * nd.nb, death);
        if (nl > 0) {
          nd.rhs_ld = nd.ld;
          nd.rhs_off = take(int64_t(nd.rhs_ld) * nl, death);
        }
      }
      if (nd.factors) {
        nd.ldq = int(align_up(nd.jn, 8));
        nd.ldf = int(align_up(nd.nb, 8));
        nd.q1_off = take(int64_t(nd.ldq) * nd.ell, death);
        nd.q2_off = take(int64_t(nd.ldq) * nd.ell, death);
        nd.rt_off = take(int64_t(nd.ldf) * nd.ell, death);
        nd.lk_off = take(int64_t(nd.ldf) * nd.ell, death);
        nd.om_off = take(int64_t(nd.ldf) * (nd.ell + 4), w + 1);  // + kProbes range-finder probes
        nd.y1_off = take(int64_t(nd.ldq) * (nd.ell + 4), w + 1);
        nd.y2_off = take(int64_t(nd.ldq) * (nd.ell + 4), w + 1);
        // K-slices of the sketches (K = nb >> jn): enough CTAs for ~2 per SM, >= 256 per slice
        const int tiles = ((nd.jn + 127) / 128) * ((nd.ell + 4 + 63) / 64);
        int S = std::max(1, std::min(8, (2 * 148 + std::max(nfac, 1) * tiles - 1) / (std::max(nfac, 1) * tiles)));
        while (S > 1 && nd.nb / S < 256) --S;
        if (sketch_split_off()) S = 1;
        nd.ysplit = S;
        if (S > 1) nd.ysp_off = take(int64_t(S - 1) * 2 * nd.ldq * (nd.ell + 4), w + 1);
      }
    }
  }
  const int64_t off = arena.end;
  P.arena_peak_bytes = 8 * off;
  P.arena_sum_bytes = 8 * sum;
  P.arena_doubles = std::max<int64_t>(off, 32);
  P.piv_ints = std::max<int64_t>(poff, 4);
  return P;
}

}  // namespace dtnb
