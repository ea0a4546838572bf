// host_sao.cpp -- host-side verification, stage 1: the
// spatial-angular-order filter of the reference (sao_filter,
// verify.cpp:303-341) with the same results, made fast where the reference
// is quadratic.
//
// The reference triangulates each image side's matched keypoints with a
// Bowyer-Watson insertion that tests every live triangle against every new
// point (verify.cpp:47-107): O(m^2) in-circle tests, 0.36 s for one 8k pair
// (SURVEY Appendix A P4).  Here the same insertion sequence runs with
// triangle adjacency: the new point is located by walking across edges from
// the last triangle created, and its cavity -- the triangles whose
// circumcircle strictly contains it -- is grown from there across edges.
// Triangles keep the reference's vertex order (make_ccw of the cavity-edge
// pair (min, max) and the point, verify.cpp:26-29, 92), and the orientation
// and in-circle predicates are evaluated with the reference's expressions in
// the same order (verify.cpp:21-43), so every decision is the same double
// computation as the reference's.  The cavity of a point inside the
// triangulation is connected (the bad triangles form a star around it); the
// first time that does not hold -- the walk fails, the located triangle is
// not bad, or the grown cavity has a boundary edge not strictly facing the
// point (badly conditioned input, e.g. a tight cluster inside a frame 10^8
// times larger, where the super triangle's predicates are pure rounding) --
// that insertion and every later one run the reference's full scan and edge
// counting verbatim.  The triangle SET after each insertion, hence the
// adjacency, equals the reference's (tested against the compiled reference
// on random, clustered, lattice, duplicated, collinear, multi-scale and real
// synthetic-scene keypoints: tests/test_sao.py).
//
// The rest -- the Delaunay-ring k nearest (verify.cpp:135-196), the angular
// order (:198-225), the cyclic edit distance (:230-255) and the per-match
// score (:303-341) -- restate the reference's definitions.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numbers>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/bandmatch_gpu.h"

namespace bmg {
void set_last_error(const std::string& msg);

namespace {

struct Pt {
  double x, y;
};

// orient2d and in_circumcircle, verify.cpp:21-43 (same expressions, same
// evaluation order: the results are bit-identical)
double orient2d(const Pt& a, const Pt& b, const Pt& c) {
  return (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
}

bool in_circumcircle(const Pt& a, const Pt& b, const Pt& c, const Pt& d) {
  const double adx = a.x - d.x, ady = a.y - d.y;
  const double bdx = b.x - d.x, bdy = b.y - d.y;
  const double cdx = c.x - d.x, cdy = c.y - d.y;
  const double ad = adx * adx + ady * ady;
  const double bd = bdx * bdx + bdy * bdy;
  const double cd = cdx * cdx + cdy * cdy;
  const double det = adx * (bdy * cd - bd * cdy) - ady * (bdx * cd - bd * cdx) + ad * (bdx * cdy - bdy * cdx);
  return det > 0.0;
}

#ifndef BMG_SAO_MAX_SPREAD
#define BMG_SAO_MAX_SPREAD 1e6
#endif
constexpr double kMaxSpread = BMG_SAO_MAX_SPREAD;

// distance of the closest pair of the first n points: a flat grid of ~n
// cells (points bucketed by a counting sort), each point against the points
// of the rings of cells around it, widening until a ring lies beyond the
// best distance found (the input has no duplicates here)
double closest_pair(const std::vector<Pt>& p, int n) {
  double lo_x = p[0].x, hi_x = p[0].x, lo_y = p[0].y, hi_y = p[0].y;
  for (int i = 0; i < n; ++i) {
    lo_x = std::min(lo_x, p[i].x);
    hi_x = std::max(hi_x, p[i].x);
    lo_y = std::min(lo_y, p[i].y);
    hi_y = std::max(hi_y, p[i].y);
  }
  const double w = std::max(hi_x - lo_x, hi_y - lo_y);
  if (!(w > 0.0)) return 0.0;
  const int g = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(n))));
  const double cell = w / g * (1.0 + 1e-9);
  auto cxy = [&](const Pt& q, int& cx, int& cy) {
    cx = std::min(g - 1, std::max(0, static_cast<int>((q.x - lo_x) / cell)));
    cy = std::min(g - 1, std::max(0, static_cast<int>((q.y - lo_y) / cell)));
  };
  std::vector<int> start(static_cast<size_t>(g) * g + 1, 0), order(n), cell_of(n);
  for (int i = 0; i < n; ++i) {
    int cx, cy;
    cxy(p[i], cx, cy);
    cell_of[i] = cy * g + cx;
    ++start[cell_of[i] + 1];
  }
  for (size_t c = 1; c < start.size(); ++c) start[c] += start[c - 1];
  {
    std::vector<int> pos(start.begin(), start.end() - 1);
    for (int i = 0; i < n; ++i) order[pos[cell_of[i]]++] = i;
  }
  double best2 = std::numeric_limits<double>::infinity();  // squared
  for (int i = 0; i < n; ++i) {
    int cx, cy;
    cxy(p[i], cx, cy);
    for (int rr = 1;; ++rr) {
      for (int dy = -rr; dy <= rr; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g) continue;
        for (int dx = -rr; dx <= rr; ++dx) {
          if (rr > 1 && std::max(std::abs(dx), std::abs(dy)) != rr) continue;
          const int x = cx + dx;
          if (x < 0 || x >= g) continue;
          const int c = y * g + x;
          for (int k = start[c]; k < start[c + 1]; ++k) {
            const int j = order[k];
            if (j == i) continue;
            const double ddx = p[i].x - p[j].x, ddy = p[i].y - p[j].y;
            best2 = std::min(best2, ddx * ddx + ddy * ddy);
          }
        }
      }
      // every cell within rr of p's has been seen: an unseen point is more
      // than rr cells' width away
      if (best2 <= (rr * cell) * (rr * cell) || rr > g + 1) break;
    }
  }
  return std::sqrt(best2);
}

// neighbour lists of the points (CSR): v's are nbr[off[v] .. off[v+1])
struct Adjacency {
  std::vector<int> off, nbr;
  bool empty() const { return off.empty(); }
};

// Bowyer-Watson with adjacency.  Triangle t has vertices v[0..2] in the
// reference's order and nb[k] = the triangle across edge (v[k], v[k+1]).
class Triangulation {
 public:
  explicit Triangulation(const std::vector<Pt>& pts_in) : n_(static_cast<int>(pts_in.size())), pts_(pts_in) {}

  // adjacency of the input points (empty when no triangle of real points
  // survives), verify.cpp:47-107
  Adjacency run() {
    if (n_ < 3) return {};
    double lo_x = pts_[0].x, hi_x = pts_[0].x, lo_y = pts_[0].y, hi_y = pts_[0].y;
    for (const Pt& p : pts_) {
      lo_x = std::min(lo_x, p.x);
      hi_x = std::max(hi_x, p.x);
      lo_y = std::min(lo_y, p.y);
      hi_y = std::max(hi_y, p.y);
    }
    const double cx = 0.5 * (lo_x + hi_x), cy = 0.5 * (lo_y + hi_y);
    const double extent = std::max({hi_x - lo_x, hi_y - lo_y, 1.0});
    const double r = 1e4 * extent;
    pts_.push_back({cx - 2.0 * r, cy - r});
    pts_.push_back({cx + 2.0 * r, cy - r});
    pts_.push_back({cx, cy + 2.0 * r});
    tris_.reserve(static_cast<size_t>(8) * n_ + 16);
    add_tri(n_, n_ + 1, n_ + 2);
    // point location starts from a triangle created near the point (a
    // coarse grid of the last triangle made in each cell): the insertion
    // order is the matches' order, spatially random, and a walk from the
    // previous insertion would cross O(sqrt n) triangles.  Only the walk's
    // start changes, not the triangle it finds.
    grid_n_ = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(n_) / 2.0)));
    grid_x0_ = lo_x;
    grid_y0_ = lo_y;
    grid_sx_ = grid_n_ / std::max(hi_x - lo_x, 1e-300);
    grid_sy_ = grid_n_ / std::max(hi_y - lo_y, 1e-300);
    grid_.assign(static_cast<size_t>(grid_n_) * grid_n_, -1);
    vert_tri_.assign(n_ + 3, -1);
    vert_tri_[n_] = vert_tri_[n_ + 1] = vert_tri_[n_ + 2] = 0;
    // ill-conditioned input (the closest pair more than kMaxSpread times
    // smaller than the extent): the in-circle decisions near the super
    // triangle are dominated by rounding, the bad set need not be a connected
    // star, so the reference's scan runs from the start
    exact_ = closest_pair(pts_, n_) * kMaxSpread < extent;
    for (int i = 0; i < n_; ++i) insert(i);

    // the edge graph of the triangles of real points, as sorted, unique
    // neighbour lists (CSR)
    Adjacency adj;
    adj.off.assign(n_ + 1, 0);
    bool any_real = false;
    auto each = [&](auto&& f) {
      for (const Tri& t : tris_)
        if (t.alive && t.v[0] < n_ && t.v[1] < n_ && t.v[2] < n_) f(t.v[0], t.v[1], t.v[2]);
      for (const V3& t : soup_)
        if (t.a < n_ && t.b < n_ && t.c < n_) f(t.a, t.b, t.c);
    };
    each([&](int a, int b, int c) {
      any_real = true;
      adj.off[a + 1] += 2;
      adj.off[b + 1] += 2;
      adj.off[c + 1] += 2;
    });
    if (!any_real) return {};
    for (int v = 0; v < n_; ++v) adj.off[v + 1] += adj.off[v];
    adj.nbr.resize(adj.off[n_]);
    std::vector<int> fill(adj.off.begin(), adj.off.end() - 1);
    each([&](int a, int b, int c) {
      adj.nbr[fill[a]++] = b;
      adj.nbr[fill[a]++] = c;
      adj.nbr[fill[b]++] = a;
      adj.nbr[fill[b]++] = c;
      adj.nbr[fill[c]++] = a;
      adj.nbr[fill[c]++] = b;
    });
    int w = 0;
    for (int v = 0; v < n_; ++v) {
      int* b = adj.nbr.data() + adj.off[v];
      int* e = adj.nbr.data() + adj.off[v + 1];
      std::sort(b, e);
      e = std::unique(b, e);
      adj.off[v] = w;
      for (int* q = b; q < e; ++q) adj.nbr[w++] = *q;
    }
    adj.off[n_] = w;
    adj.nbr.resize(w);
    return adj;
  }

 private:
  struct Tri {
    int v[3];
    int nb[3];
    bool alive;
    int mark;  // insertion that marked it bad / visited
  };

  // make_ccw (verify.cpp:26-29)
  int add_tri(int a, int b, int c) {
    if (orient2d(pts_[a], pts_[b], pts_[c]) < 0.0) std::swap(b, c);
    tris_.push_back(Tri{{a, b, c}, {-1, -1, -1}, true, -1});
    const int t = static_cast<int>(tris_.size()) - 1;
    if (!vert_tri_.empty()) vert_tri_[a] = vert_tri_[b] = vert_tri_[c] = t;
    return t;
  }

  bool bad(int t, int i) {
    const Tri& T = tris_[t];
    return in_circumcircle(pts_[T.v[0]], pts_[T.v[1]], pts_[T.v[2]], pts_[i]);
  }

  // a live triangle containing point i (or -1): walk from the last created
  // triangle, crossing an edge that has the point strictly on its outer side
  int cell_of(const Pt& p) const {
    const double top = grid_n_ - 1;
    double fx = (p.x - grid_x0_) * grid_sx_, fy = (p.y - grid_y0_) * grid_sy_;
    fx = fx >= 0.0 ? std::min(fx, top) : 0.0;  // also NaN -> 0
    fy = fy >= 0.0 ? std::min(fy, top) : 0.0;
    return static_cast<int>(fy) * grid_n_ + static_cast<int>(fx);
  }

  // a live triangle to start the walk for point p: one incident to an
  // already inserted vertex in p's cell or the nearest non-empty ring of
  // cells around it (every inserted vertex keeps a live incident triangle:
  // a cavity's vertices all lie on its boundary and get new triangles)
  int walk_start(const Pt& p) const {
    if (grid_.empty()) return last_;
    const int c = cell_of(p), cx = c % grid_n_, cy = c / grid_n_;
    for (int rr = 0; rr < grid_n_; ++rr) {
      for (int dy = -rr; dy <= rr; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= grid_n_) continue;
        for (int dx = -rr; dx <= rr; ++dx) {
          if (std::max(std::abs(dx), std::abs(dy)) != rr) continue;
          const int x = cx + dx;
          if (x < 0 || x >= grid_n_) continue;
          const int v = grid_[y * grid_n_ + x];
          if (v >= 0 && vert_tri_[v] >= 0 && tris_[vert_tri_[v]].alive) return vert_tri_[v];
        }
      }
      if (rr >= 3) break;  // sparse early insertions: the last triangle made
    }
    return last_;
  }

  int locate(int i) {
    const Pt& p = pts_[i];
    int t = walk_start(p);
    for (int steps = 0; steps < 4 * static_cast<int>(tris_.size()) + 16; ++steps) {
      const Tri& T = tris_[t];
      // the triangle's own winding (make_ccw leaves collinear triples as given)
      const double w = orient2d(pts_[T.v[0]], pts_[T.v[1]], pts_[T.v[2]]);
      if (w <= 0.0) return -1;
      int next = -1;
      const int k0 = steps % 3;
      for (int kk = 0; kk < 3; ++kk) {
        const int k = (k0 + kk) % 3;
        if (orient2d(pts_[T.v[k]], pts_[T.v[(k + 1) % 3]], p) < 0.0) {
          next = T.nb[k];
          break;
        }
      }
      if (next < 0) {
        // inside (or on the boundary of) T, or outside the super triangle
        for (int k = 0; k < 3; ++k)
          if (orient2d(pts_[T.v[k]], pts_[T.v[(k + 1) % 3]], p) < 0.0) return -1;
        return t;
      }
      t = next;
    }
    return -1;
  }

  void insert(int i) {
    if (!exact_ && fast_insert(i)) return;
    exact_ = true;
    scan_insert(i);
  }

  // The reference's insertion (verify.cpp:76-93): every live triangle whose
  // circumcircle strictly contains the point is removed; edges appearing
  // once among them are joined to the point.  Used from the first insertion
  // whose cavity does not look like a clean star around the point on (badly
  // conditioned input); neighbour links are no longer kept then.
  void scan_insert(int i) {
    if (soup_.empty()) {  // entering scan mode: the live triangles, no links
      for (const Tri& T : tris_)
        if (T.alive) soup_.push_back({T.v[0], T.v[1], T.v[2]});
      for (Tri& T : tris_) T.alive = false;
    }
    keep_.clear();
    keys_.clear();
    for (const V3& t : soup_) {
      if (in_circumcircle(pts_[t.a], pts_[t.b], pts_[t.c], pts_[i])) {
        const int v[3] = {t.a, t.b, t.c};
        for (int k = 0; k < 3; ++k) {
          const int a = v[k], b = v[(k + 1) % 3];
          keys_.push_back((static_cast<uint64_t>(std::min(a, b)) << 32) | static_cast<uint32_t>(std::max(a, b)));
        }
      } else {
        keep_.push_back(t);
      }
    }
    if (keys_.empty()) return;
    soup_.swap(keep_);
    std::sort(keys_.begin(), keys_.end());
    for (size_t a = 0; a < keys_.size();) {
      size_t b = a + 1;
      while (b < keys_.size() && keys_[b] == keys_[a]) ++b;
      if (b - a == 1) {
        int u = static_cast<int>(keys_[a] >> 32), v = static_cast<int>(keys_[a] & 0xffffffffu), w = i;
        if (orient2d(pts_[u], pts_[v], pts_[w]) < 0.0) std::swap(v, w);  // make_ccw
        soup_.push_back({u, v, w});
      }
      a = b;
    }
  }

  // The same insertion with adjacency: point location by walking, the
  // cavity grown across edges.  Returns false -- before changing anything --
  // when the walk fails, the located triangle is not bad, or the cavity is
  // not a star around the point (some boundary edge not strictly facing
  // it): the caller then switches to the reference's scan.
  bool fast_insert(int i) {
    cavity_.clear();
    const int start = locate(i);
    if (start < 0 || !bad(start, i)) return false;
    tris_[start].mark = i;
    cavity_.push_back(start);
    for (size_t q = 0; q < cavity_.size(); ++q) {
      const Tri& T = tris_[cavity_[q]];
      for (int k = 0; k < 3; ++k) {
        const int u = T.nb[k];
        if (u < 0 || tris_[u].mark == i) continue;
        tris_[u].mark = i;  // visited (bad or not) for this insertion
        if (bad(u, i)) cavity_.push_back(u);
      }
    }
    for (int t : cavity_) tris_[t].mark = -2 - i;  // cavity members
    // boundary edges: edges of cavity triangles whose neighbour is outside
    edges_.clear();
    for (int t : cavity_) {
      const Tri& T = tris_[t];
      for (int k = 0; k < 3; ++k) {
        const int u = T.nb[k];
        if (u >= 0 && tris_[u].mark == -2 - i) continue;  // interior edge
        const int a = T.v[k], b = T.v[(k + 1) % 3];
        if (!(orient2d(pts_[a], pts_[b], pts_[i]) > 0.0)) {
          for (int c : cavity_) tris_[c].mark = -1;
          return false;
        }
        edges_.push_back({a, b, u});
      }
    }
    for (int t : cavity_) tris_[t].alive = false;
    // new triangles make_ccw(min, max, i) (verify.cpp:91-92), linked to the
    // outside triangle across the cavity edge and to each other across the
    // edges through i
    spoke_.clear();
    for (const auto& e : edges_) {
      const int lo = std::min(e.a, e.b), hi = std::max(e.a, e.b);
      const int t = add_tri(lo, hi, i);
      Tri& T = tris_[t];
      for (int k = 0; k < 3; ++k) {
        const int a = T.v[k], b = T.v[(k + 1) % 3];
        if ((a == lo && b == hi) || (a == hi && b == lo)) {
          T.nb[k] = e.outside;
          if (e.outside >= 0) {
            Tri& O = tris_[e.outside];
            for (int j = 0; j < 3; ++j) {
              const int oa = O.v[j], ob = O.v[(j + 1) % 3];
              if ((oa == lo && ob == hi) || (oa == hi && ob == lo)) O.nb[j] = t;
            }
          }
        } else {
          const int other = a == i ? b : a;  // the edge (other, i)
          size_t f = 0;
          while (f < spoke_.size() && spoke_[f].v != other) ++f;
          if (f == spoke_.size()) {
            spoke_.push_back({other, t, k});
          } else {
            T.nb[k] = spoke_[f].t;
            tris_[spoke_[f].t].nb[spoke_[f].k] = t;
          }
        }
      }
      last_ = t;
    }
    if (!grid_.empty()) grid_[cell_of(pts_[i])] = i;
    return true;
  }

  struct EdgeRec {
    int a, b, outside;
  };
  struct V3 {
    int a, b, c;
  };
  std::vector<V3> soup_, keep_;  // scan mode: the live triangles, as the reference keeps them
  std::vector<uint64_t> keys_;
  bool exact_ = false;
  std::vector<EdgeRec> edges_;
  struct Spoke {
    int v, t, k;  // edge (v, new point) of triangle t, its index k
  };
  std::vector<Spoke> spoke_;  // the cavity's new spokes (a handful per insertion)
  std::vector<int> grid_;     // per cell: the last vertex inserted there
  std::vector<int> vert_tri_; // per vertex: a live incident triangle
  int grid_n_ = 0;
  double grid_x0_ = 0, grid_y0_ = 0, grid_sx_ = 0, grid_sy_ = 0;
  int n_;
  std::vector<Pt> pts_;
  std::vector<Tri> tris_;
  std::vector<int> cavity_;
  int last_ = 0;
};

double dist2(const Pt& a, const Pt& b) {
  const double dx = a.x - b.x, dy = a.y - b.y;
  return dx * dx + dy * dy;
}

// ring members by (squared distance, index), verify.cpp:117-124
void by_distance(const Pt& c, const std::vector<Pt>& pts, std::vector<int>& ring) {
  std::sort(ring.begin(), ring.end(), [&](int u, int v) {
    const double du = dist2(c, pts[u]), dv = dist2(c, pts[v]);
    if (du != dv) return du < dv;
    return u < v;
  });
}

// knn_from_delaunay, verify.cpp:135-196: rings of the triangulation's edge
// graph around each point, nearer rings first; plain nearest neighbours when
// the set has duplicates or cannot be triangulated
std::vector<std::vector<int>> delaunay_knn(const std::vector<Pt>& pts, int k, bool* fallback) {
  const int n = static_cast<int>(pts.size());
  std::vector<std::vector<int>> out(n);
  *fallback = false;
  if (k == 0 || n <= 1) return out;
  bool dup = false;
  {
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int u, int v) {
      if (pts[u].x != pts[v].x) return pts[u].x < pts[v].x;
      return pts[u].y < pts[v].y;
    });
    for (int i = 0; i + 1 < n; ++i)
      if (pts[order[i]].x == pts[order[i + 1]].x && pts[order[i]].y == pts[order[i + 1]].y) dup = true;
  }
  Adjacency adj;
  if (!dup) adj = Triangulation(pts).run();
  if (adj.empty()) {
    *fallback = true;
    for (int i = 0; i < n; ++i) {
      std::vector<int> others;
      others.reserve(n - 1);
      for (int j = 0; j < n; ++j)
        if (j != i) others.push_back(j);
      by_distance(pts[i], pts, others);
      if (static_cast<int>(others.size()) > k) others.resize(k);
      out[i] = std::move(others);
    }
    return out;
  }
  std::vector<int> visited(n, -1), frontier, ring;
  for (int i = 0; i < n; ++i) {
    std::vector<int>& res = out[i];
    visited[i] = i;
    frontier.assign(1, i);
    while (static_cast<int>(res.size()) < k && !frontier.empty()) {
      ring.clear();
      for (int u : frontier)
        for (int e = adj.off[u]; e < adj.off[u + 1]; ++e) {
          const int v = adj.nbr[e];
          if (visited[v] != i) {
            visited[v] = i;
            ring.push_back(v);
          }
        }
      by_distance(pts[i], pts, ring);
      res.insert(res.end(), ring.begin(), ring.end());
      frontier.swap(ring);
    }
    if (static_cast<int>(res.size()) > k) res.resize(k);
    if (static_cast<int>(res.size()) < k) {
      std::vector<int> rest;
      for (int j = 0; j < n; ++j)
        if (visited[j] != i) rest.push_back(j);
      by_distance(pts[i], pts, rest);
      for (int j : rest) {
        if (static_cast<int>(res.size()) >= k) break;
        res.push_back(j);
      }
    }
  }
  return out;
}

// angular_order, verify.cpp:198-225 (atan2 in [0, 2 pi), then distance, index)
std::vector<int> angular(const Pt& c, const std::vector<int>& nbrs, const std::vector<Pt>& pts) {
  struct Key {
    double angle, d2;
    int idx;
  };
  std::vector<Key> keys;
  keys.reserve(nbrs.size());
  for (int idx : nbrs) {
    const double dx = pts[idx].x - c.x, dy = pts[idx].y - c.y;
    double a = std::atan2(dy, dx);
    if (a < 0.0) a += 2.0 * std::numbers::pi;
    keys.push_back({a, dx * dx + dy * dy, idx});
  }
  std::sort(keys.begin(), keys.end(), [](const Key& u, const Key& v) {
    if (u.angle != v.angle) return u.angle < v.angle;
    if (u.d2 != v.d2) return u.d2 < v.d2;
    return u.idx < v.idx;
  });
  std::vector<int> out;
  out.reserve(keys.size());
  for (const Key& k : keys) out.push_back(k.idx);
  return out;
}

// cyclic_edit_distance, verify.cpp:230-255: min over rotations of b of the
// Levenshtein distance
int cyclic_edit(const std::vector<int>& a, const std::vector<int>& b) {
  if (b.empty()) return static_cast<int>(a.size());
  if (a.empty()) return static_cast<int>(b.size());
  const size_t na = a.size(), nb = b.size();
  // rows of the DP on the stack for the usual ring sizes (n_neighbors = 6);
  // b doubled so a rotation is a window (no modulo in the inner loop)
  constexpr size_t kSmall = 32;
  int prev_s[kSmall + 1], cur_s[kSmall + 1], bb_s[2 * kSmall];
  std::vector<int> prev_v, cur_v, bb_v;
  int *prev = prev_s, *cur = cur_s, *bb = bb_s;
  if (nb > kSmall) {
    prev_v.resize(nb + 1);
    cur_v.resize(nb + 1);
    bb_v.resize(2 * nb);
    prev = prev_v.data();
    cur = cur_v.data();
    bb = bb_v.data();
  }
  for (size_t j = 0; j < nb; ++j) bb[j] = bb[j + nb] = b[j];
  int best = std::numeric_limits<int>::max();
  for (size_t rot = 0; rot < nb; ++rot) {
    const int* br = bb + rot;
    for (size_t j = 0; j <= nb; ++j) prev[j] = static_cast<int>(j);
    for (size_t i = 1; i <= na; ++i) {
      cur[0] = static_cast<int>(i);
      const int ai = a[i - 1];
      for (size_t j = 1; j <= nb; ++j) {
        const int sub = prev[j - 1] + (ai == br[j - 1] ? 0 : 1);
        cur[j] = std::min({prev[j] + 1, cur[j - 1] + 1, sub});
      }
      std::swap(prev, cur);
    }
    best = std::min(best, prev[nb]);
  }
  return best;
}

// one image side (verify.cpp:265-300): positions deduplicated by exact
// coordinates (first match index labels each position), rings of labels
struct Side {
  std::vector<Pt> pos;
  std::vector<int> pos_of;
  std::vector<int> label;
  std::vector<std::vector<int>> rings;
  bool fallback = false;
};

Side side_of(const int32_t* matches, uint64_t m, bool query, const float* kps, int k) {
  Side s;
  s.pos_of.resize(m);
  struct H {
    size_t operator()(const std::pair<double, double>& p) const {
      return std::hash<double>()(p.first) * 1000003u ^ std::hash<double>()(p.second);
    }
  };
  std::unordered_map<std::pair<double, double>, int, H> seen;
  seen.reserve(m * 2);
  for (uint64_t i = 0; i < m; ++i) {
    const int idx = matches[2 * i + (query ? 0 : 1)];
    const std::pair<double, double> key(kps[4 * static_cast<size_t>(idx)], kps[4 * static_cast<size_t>(idx) + 1]);
    const auto [it, inserted] = seen.emplace(key, static_cast<int>(s.pos.size()));
    if (inserted) {
      s.pos.push_back({key.first, key.second});
      s.label.push_back(static_cast<int>(i));
    }
    s.pos_of[i] = it->second;
  }
  const std::vector<std::vector<int>> knn = delaunay_knn(s.pos, k, &s.fallback);
  s.rings.resize(m);
  for (uint64_t i = 0; i < m; ++i) {
    const int p = s.pos_of[i];
    for (int q : angular(s.pos[p], knn[p], s.pos)) s.rings[i].push_back(s.label[q]);
  }
  return s;
}

}  // namespace
}  // namespace bmg

using namespace bmg;

extern "C" {

int bmg_delaunay_knn(const double* xy, uint64_t n, int k, int32_t* neighbors_out, int* fallback_out) {
  if ((n && !xy) || (n && k > 0 && !neighbors_out) || !fallback_out || k < 0) {
    set_last_error(k < 0 ? "n_neighbors must be non-negative" : "null argument");
    return BMG_INVALID_ARGUMENT;
  }
  try {
    std::vector<Pt> pts(n);
    for (uint64_t i = 0; i < n; ++i) pts[i] = Pt{xy[2 * i], xy[2 * i + 1]};
    bool fb = false;
    const std::vector<std::vector<int>> nb = delaunay_knn(pts, k, &fb);
    for (uint64_t i = 0; i < n; ++i)
      for (int j = 0; j < k; ++j)
        neighbors_out[i * k + j] = j < static_cast<int>(nb[i].size()) ? nb[i][j] : -1;
    *fallback_out = fb ? 1 : 0;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return BMG_OUT_OF_MEMORY;
  }
  return BMG_OK;
}

int bmg_sao_filter(const int32_t* matches, uint64_t n_matches, const float* query_kps, uint64_t n_query,
                   const float* train_kps, uint64_t n_train, int n_neighbors, double score_threshold,
                   uint8_t* keep_out, double* scores_out, uint32_t* flags_out) {
  if ((n_matches && !matches) || !keep_out || !scores_out || !flags_out) {
    set_last_error("null argument");
    return BMG_INVALID_ARGUMENT;
  }
  // verify.cpp:305-313
  if (n_neighbors < 1) {
    set_last_error("n_neighbors must be >= 1");
    return BMG_INVALID_ARGUMENT;
  }
  if (!(score_threshold >= 0.0)) {
    set_last_error("score_threshold must be non-negative");
    return BMG_INVALID_ARGUMENT;
  }
  for (uint64_t i = 0; i < n_matches; ++i) {
    const int32_t q = matches[2 * i], t = matches[2 * i + 1];
    if (q < 0 || static_cast<uint64_t>(q) >= n_query || t < 0 || static_cast<uint64_t>(t) >= n_train) {
      set_last_error("match index outside its keypoint list");
      return BMG_INVALID_ARGUMENT;
    }
  }
  *flags_out = 0;
  for (uint64_t i = 0; i < n_matches; ++i) scores_out[i] = 0.0;
  if (n_matches < static_cast<uint64_t>(n_neighbors) + 1) {  // :321-325
    for (uint64_t i = 0; i < n_matches; ++i) keep_out[i] = 1;
    *flags_out = BMG_SAO_PASSTHROUGH;
    return BMG_OK;
  }
  try {
    const Side q = side_of(matches, n_matches, true, query_kps, n_neighbors);
    const Side t = side_of(matches, n_matches, false, train_kps, n_neighbors);
    if (q.fallback || t.fallback) *flags_out |= BMG_SAO_DELAUNAY_FALLBACK;
    for (uint64_t i = 0; i < n_matches; ++i) {
      const std::vector<int>& rq = q.rings[i];
      const std::vector<int>& rt = t.rings[i];
      const size_t len = std::max(rq.size(), rt.size());
      scores_out[i] = len == 0 ? 0.0 : cyclic_edit(rq, rt) / static_cast<double>(len);
      keep_out[i] = scores_out[i] <= score_threshold ? 1 : 0;
    }
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return BMG_OUT_OF_MEMORY;
  }
  return BMG_OK;
}

}  // extern "C"
