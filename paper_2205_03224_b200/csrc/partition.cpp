// Multilevel p-way vertex-separator reordering (Alg. 3 pGeMSLRReordering,
// P:L582-597) and RCM ordering of the last separator.
//
// Level l partitions the induced subgraph of |C_{l-1}| + |C_{l-1}^T| (the
// previous separator; C_{-1} = A) into p parts by recursive bisection —
// coordinate bisection when vertex coordinates are supplied, BFS level-set
// bisection from a pseudo-peripheral vertex otherwise (reading Q23: ParMETIS is
// not available).  The vertex separator is a vertex cover of the cut edges: a
// vertex joins it when it has a neighbour in a part of HIGHER id, so no edge
// joins two different parts.  The recursion stops at l_ev levels
// or when the separator has fewer than 2p vertices (reading Q24).
#include <algorithm>
#include <numeric>
#include <queue>

#include "plan.hpp"

namespace gemslr {

Graph build_graph(int64_t n, const int64_t *rowptr, const int32_t *colidx) {
  Graph g;
  g.n = n;
  std::vector<int64_t> deg(n, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      int64_t j = colidx[p];
      if (j == i) continue;
      deg[i]++;
      deg[j]++;
    }
  std::vector<int64_t> ptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + deg[i];
  std::vector<int32_t> adj(ptr[n]);
  std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      int64_t j = colidx[p];
      if (j == i) continue;
      adj[pos[i]++] = (int32_t)j;
      adj[pos[j]++] = (int32_t)i;
    }
  // sort + unique each row (pattern of A + A^T)
  g.ptr.assign(n + 1, 0);
  g.adj.reserve(adj.size());
  for (int64_t i = 0; i < n; ++i) {
    auto b = adj.begin() + ptr[i], e = adj.begin() + ptr[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    g.adj.insert(g.adj.end(), b, u);
    g.ptr[i + 1] = (int64_t)g.adj.size();
  }
  return g;
}

namespace {

// BFS over the induced subgraph (mask `in` == stamp) from `start`; returns the
// order and writes dist.  Neighbours are visited in ascending index order.
int64_t bfs(const Graph &g, const std::vector<int32_t> &in, int32_t stamp, int32_t start,
            std::vector<int32_t> &dist, std::vector<int32_t> &order) {
  order.clear();
  order.push_back(start);
  dist[start] = 0;
  int64_t maxd = 0;
  for (size_t h = 0; h < order.size(); ++h) {
    int32_t v = order[h];
    for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
      int32_t u = g.adj[p];
      if (in[u] != stamp || dist[u] >= 0) continue;
      dist[u] = dist[v] + 1;
      maxd = std::max<int64_t>(maxd, dist[u]);
      order.push_back(u);
    }
  }
  return maxd;
}

int64_t sub_degree(const Graph &g, const std::vector<int32_t> &in, int32_t stamp, int32_t v) {
  int64_t d = 0;
  for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) d += in[g.adj[p]] == stamp;
  return d;
}

// George-Liu pseudo-peripheral vertex of the component containing `start`.
int32_t pseudo_peripheral(const Graph &g, const std::vector<int32_t> &in, int32_t stamp, int32_t start,
                          std::vector<int32_t> &dist) {
  std::vector<int32_t> order;
  int32_t v = start;
  int64_t ecc = -1;
  for (int it = 0; it < 16; ++it) {
    for (int32_t u : order) dist[u] = -1;
    int64_t e = bfs(g, in, stamp, v, dist, order);
    // candidate: farthest vertex of minimum degree, ties -> lowest index
    int32_t best = -1;
    int64_t bestdeg = 0;
    for (int32_t u : order)
      if (dist[u] == e) {
        int64_t d = sub_degree(g, in, stamp, u);
        if (best < 0 || d < bestdeg || (d == bestdeg && u < best)) { best = u; bestdeg = d; }
      }
    for (int32_t u : order) dist[u] = -1;
    if (e <= ecc) break;
    ecc = e;
    v = best;
  }
  for (int32_t u : order) dist[u] = -1;
  return v;
}

struct Bisector {
  const Graph &g;
  const SetupOptions &opt;
  std::vector<int32_t> in;      // stamp mask
  std::vector<int32_t> dist;
  int32_t stamp = 0;
  Bisector(const Graph &g_, const SetupOptions &o) : g(g_), opt(o), in(g_.n, -1), dist(g_.n, -1) {}

  // Order `verts` (sorted ascending) for a bisection split.
  void split_order(std::vector<int32_t> &verts) {
    if (opt.coords && opt.coord_dim > 0) {
      // recursive coordinate bisection: axis of largest extent (ties -> lowest axis),
      // order by (coordinate, index)
      const int d = opt.coord_dim;
      int ax = 0;
      double best = -1;
      for (int a = 0; a < d; ++a) {
        double lo = 1e300, hi = -1e300;
        for (int32_t v : verts) { double c = opt.coords[(int64_t)v * d + a]; lo = std::min(lo, c); hi = std::max(hi, c); }
        if (hi - lo > best + 1e-12) { best = hi - lo; ax = a; }
      }
      std::stable_sort(verts.begin(), verts.end(), [&](int32_t a, int32_t b) {
        double ca = opt.coords[(int64_t)a * d + ax], cb = opt.coords[(int64_t)b * d + ax];
        if (ca != cb) return ca < cb;
        return a < b;
      });
      return;
    }
    // BFS level-set order from a pseudo-peripheral vertex; further components
    // start at their lowest unvisited vertex.
    ++stamp;
    for (int32_t v : verts) in[v] = stamp;
    std::vector<int32_t> out, order;
    out.reserve(verts.size());
    for (int32_t v : verts) {
      if (dist[v] >= 0) continue;
      int32_t s = pseudo_peripheral(g, in, stamp, v, dist);
      bfs(g, in, stamp, s, dist, order);
      out.insert(out.end(), order.begin(), order.end());
    }
    for (int32_t v : out) dist[v] = -1;
    verts.swap(out);
  }

  // Recursive bisection of `verts` into parts [first, first + p).
  void bisect(std::vector<int32_t> verts, int p, int first, std::vector<int32_t> &part) {
    if (p == 1) {
      for (int32_t v : verts) part[v] = first;
      return;
    }
    const int pa = p / 2;
    std::sort(verts.begin(), verts.end());
    split_order(verts);
    const size_t na = verts.size() * (size_t)pa / (size_t)p;
    std::vector<int32_t> a(verts.begin(), verts.begin() + na), b(verts.begin() + na, verts.end());
    bisect(std::move(a), pa, first, part);
    bisect(std::move(b), p - pa, first + pa, part);
  }
};

// Reverse Cuthill-McKee of the induced subgraph on `verts` (reading
// Q11): components in order of their lowest vertex, each started at a
// pseudo-peripheral vertex, neighbours by (degree, index); then reversed.
std::vector<int32_t> rcm(const Graph &g, const std::vector<int32_t> &verts) {
  std::vector<int32_t> in(g.n, -1), dist(g.n, -1);
  const int32_t stamp = 1;
  for (int32_t v : verts) in[v] = stamp;
  std::vector<char> done(g.n, 0);
  std::vector<int32_t> order;
  std::vector<int32_t> sorted(verts);
  std::sort(sorted.begin(), sorted.end());
  for (int32_t v0 : sorted) {
    if (done[v0]) continue;
    int32_t s = pseudo_peripheral(g, in, stamp, v0, dist);
    size_t head = order.size();
    order.push_back(s);
    done[s] = 1;
    while (head < order.size()) {
      int32_t v = order[head++];
      std::vector<std::pair<int64_t, int32_t>> nb;
      for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
        int32_t u = g.adj[p];
        if (in[u] != stamp || done[u]) continue;
        nb.push_back({sub_degree(g, in, stamp, u), u});
      }
      std::sort(nb.begin(), nb.end());
      for (auto &e : nb) { done[e.second] = 1; order.push_back(e.second); }
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

}  // namespace

bool build_structure(const Graph &g, const SetupOptions &opt, Structure &st, Error &err) {
  const int64_t n = g.n;
  const int p = opt.p;
  st = Structure();
  st.n = n;
  if (p > n) {
    err = {-3, "PARTITION: p = " + std::to_string(p) + " exceeds the " + std::to_string(n) + " vertices"};
    return false;
  }
  Bisector bis(g, opt);
  std::vector<int32_t> current(n);
  std::iota(current.begin(), current.end(), 0);
  std::vector<int32_t> part(n, -1);
  std::vector<char> insep(n, 0);
  st.o.push_back(0);
  int64_t pos = 0;
  for (int l = 0; l < opt.levels; ++l) {
    if (l > 0 && (int64_t)current.size() < 2 * (int64_t)p) break;   // reading Q24
    for (int32_t v : current) part[v] = -1;
    bis.bisect(current, p, 0, part);
    // vertex cover of the cut edges: v joins the separator when a neighbour in
    // the current set lies in a part of higher id
    std::vector<int32_t> sep;
    for (int32_t v : current) {
      bool s = false;
      for (int64_t q = g.ptr[v]; q < g.ptr[v + 1] && !s; ++q) {
        int32_t u = g.adj[q];
        if (part[u] >= 0 && part[u] > part[v]) s = true;
      }
      if (s) { sep.push_back(v); insep[v] = 1; }
    }
    // interiors of each part = blocks of level l.  Local ordering of B_l
    // (P:L660-662 allows a local reordering): with coordinates, the part's
    // points sorted with its LONGEST axis varying fastest (axes by decreasing
    // extent from fastest to slowest, ties -> lower axis, then index) — the
    // ILUT level-schedule depth of a 32x32x64 box drops from 563/758 (x
    // fastest) to 371/470 at the same fill.  ILU(0) depth does not depend on
    // this choice (same edge orientation), so ILU(0) and runs without
    // coordinates keep ascending index.
    std::vector<std::vector<int32_t>> members(p);
    for (int32_t v : current)
      if (!insep[v]) members[part[v]].push_back(v);
    if (opt.coords && opt.coord_dim > 0 && opt.ilu == 1) {
      const int d = opt.coord_dim;
      for (auto &mem : members) {
        if (mem.size() < 2) continue;
        std::vector<double> lo(d, 1e300), hi(d, -1e300);
        for (int32_t v : mem)
          for (int a = 0; a < d; ++a) {
            const double c = opt.coords[(int64_t)v * d + a];
            lo[a] = std::min(lo[a], c);
            hi[a] = std::max(hi[a], c);
          }
        std::vector<int> ax(d);
        std::iota(ax.begin(), ax.end(), 0);
        // slowest first: increasing extent (ties -> higher axis slower so x stays fastest among equals)
        std::stable_sort(ax.begin(), ax.end(), [&](int a, int b) { return hi[a] - lo[a] < hi[b] - lo[b] - 1e-12; });
        std::reverse(ax.begin(), ax.end());      // now: fastest (longest) first
        std::sort(mem.begin(), mem.end(), [&](int32_t a, int32_t b) {
          for (int i = d - 1; i >= 0; --i) {     // compare slowest axis first
            const double ca = opt.coords[(int64_t)a * d + ax[i]], cb = opt.coords[(int64_t)b * d + ax[i]];
            if (ca != cb) return ca < cb;
          }
          return a < b;
        });
      }
    }
    // Boundary rows last (a local reordering of B_l; DESIGN 6b): the rows of
    // a block adjacent to a later level (E_l's columns, F_l's rows) go after its interior
    // rows.  Since L is lower and U upper triangular, z1 at those rows then needs only
    // the U sweep over them (the DOWN's U sweep shrinks to this tail) and L^-1 F_l y2 is
    // zero before them (the UP's L sweep shrinks to it too; Alg. 2 is unchanged up to
    // rounding, the oracle follows it literally).  The tail is coloured greedily (a
    // colour per vertex, distinct from every tail vertex within opt.tail_dist tail edges,
    // in the order above) and sorted by colour, which keeps the level-schedule depth of
    // the tail sweeps small (C5 level 0, 32x32x64: U tail 95, L tail 14 levels).
    if (opt.tail) {
      std::vector<int32_t> colr(n, -1), seenv(n, -1);
      for (auto &mem : members) {
        std::vector<int32_t> head, tl;
        for (int32_t v : mem) {
          bool b = false;
          for (int64_t q = g.ptr[v]; q < g.ptr[v + 1] && !b; ++q) b = insep[g.adj[q]] != 0;
          (b ? tl : head).push_back(v);
        }
        if (tl.empty()) continue;
        for (int32_t v : tl) colr[v] = -2;                         // tail, not yet coloured
        std::vector<int32_t> fr, fr2, used;
        for (int32_t v : tl) {
          fr.assign(1, v);
          seenv[v] = v;
          used.clear();
          for (int d = 0; d < opt.tail_dist && !fr.empty(); ++d) {
            fr2.clear();
            for (int32_t u : fr)
              for (int64_t q = g.ptr[u]; q < g.ptr[u + 1]; ++q) {
                const int32_t w = g.adj[q];
                if (colr[w] == -1 || seenv[w] == v) continue;      // not in this tail, or seen
                seenv[w] = v;
                fr2.push_back(w);
                if (colr[w] >= 0) used.push_back(colr[w]);
              }
            fr.swap(fr2);
          }
          std::sort(used.begin(), used.end());
          int c = 0;
          for (int32_t x : used)
            if (x == c) ++c;
            else if (x > c) break;
          colr[v] = c;
        }
        std::stable_sort(tl.begin(), tl.end(), [&](int32_t a, int32_t b) { return colr[a] < colr[b]; });
        for (int32_t v : tl) colr[v] = -1;
        mem = head;
        mem.insert(mem.end(), tl.begin(), tl.end());
      }
    }
    std::vector<int64_t> bl{pos};
    for (int q = 0; q < p; ++q) {
      for (int32_t v : members[q]) st.perm.push_back(v);
      pos += (int64_t)members[q].size();
      bl.push_back(pos);
    }
    st.blk.push_back(bl);
    st.o.push_back(pos);
    for (int32_t v : current) part[v] = -1;
    for (int32_t v : sep) insep[v] = 0;
    current.swap(sep);
    st.L = l + 1;
  }
  // C_{l_ev-1}: RCM order, then near-equal contiguous blocks
  std::vector<int32_t> order = rcm(g, current);
  for (int32_t v : order) st.perm.push_back(v);
  const int64_t s = (int64_t)order.size();
  int nlast = opt.last_blocks > 0 ? opt.last_blocks : p;
  if (nlast > s) nlast = (int)s;
  st.last.push_back(pos);
  for (int q = 1; q <= nlast; ++q) st.last.push_back(pos + s * q / nlast);
  st.iperm.assign(n, -1);
  for (int64_t i = 0; i < n; ++i) st.iperm[st.perm[i]] = i;
  return true;
}

}  // namespace gemslr
