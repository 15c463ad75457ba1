// linkage.cu — the reference's fixed linkage model (bounded) FLT without the
// n x n similarity matrix: learn_tree_upgma (linkage.hpp:133-264) over the
// problem-structure similarity vig_similarity / weight_similarity
// (linkage.hpp:102-119), which is non-zero only on the graph's edges.
//
// learn_tree_upgma repeatedly merges the allowed pair of clusters (merged size
// <= bound) with the highest mean inter-cluster similarity sum/(|A||B|), ties
// to the lexicographically smallest pair of representatives (min variable),
// the merged cluster keeping the smaller representative's slot and sum(A+B, D)
// = sum(A, D) + sum(B, D).  With a sparse similarity every pair is either
// adjacent (positive sum) or has score 0, so the same sequence of merges is:
//   1. while an allowed positive pair exists: the best of them (a lazy-deleted
//      heap of adjacent pairs, compared exactly like score_less /
//      candidate_before, sums accumulated in the reference's order);
//   2. then score-0 merges in lexicographic order of representatives: the
//      smallest representative x that has an allowed partner, with the
//      smallest such partner (a segment tree of cluster sizes over
//      representatives).  Merges only grow clusters, so no positive pair
//      becomes allowed again in phase 2.
// Memory and time are O((n + q) log n) instead of O(n^2) / O(n^3): bounded FLT
// models for 10^6-vertex instances.  Output: singletons in variable order,
// then the merged sets in merge order, the full set never emitted (Fos,
// linkage.hpp:121-131).
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <limits>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "gomix_gpu.h"
#include "internal.cuh"

using namespace gomix_b200;

namespace {

struct Cand {
  double sum, w;  // score = sum / w
  uint32_t ka, kb;  // representatives, ka < kb
  uint32_t va, vb;  // versions of clusters ka, kb when pushed
};

// true when x should be merged before y (candidate_before, linkage.hpp:185-191)
bool before(const Cand& x, const Cand& y) {
  if (y.sum * x.w < x.sum * y.w) return true;
  if (x.sum * y.w < y.sum * x.w) return false;
  return x.ka != y.ka ? x.ka < y.ka : x.kb < y.kb;
}

struct HeapOrder {
  bool operator()(const Cand& x, const Cand& y) const { return before(y, x); }
};

struct Flt {
  uint64_t n = 0, bound = 0;
  std::vector<uint8_t> alive;
  std::vector<uint64_t> size;
  std::vector<uint32_t> version;
  std::vector<std::vector<uint32_t>> members;
  std::vector<std::unordered_map<uint32_t, double>> adj;  // cluster (rep) -> similarity sum
  std::vector<std::vector<uint32_t>> sets;                // merged sets in merge order
  uint64_t remaining = 0;

  void merge(uint32_t a, uint32_t b) {  // a < b: a keeps its slot (the smaller representative)
    std::vector<uint32_t> m;
    m.reserve(members[a].size() + members[b].size());
    std::merge(members[a].begin(), members[a].end(), members[b].begin(), members[b].end(), std::back_inserter(m));
    members[a] = std::move(m);
    members[b].clear();
    members[b].shrink_to_fit();
    alive[b] = 0;
    size[a] += size[b];
    ++version[a];
    ++version[b];
    if (size[a] < n) sets.push_back(members[a]);
    --remaining;
    // sum(A+B, D) = sum(A, D) + sum(B, D), in that order (linkage.hpp:247-251)
    auto& A = adj[a];
    auto& Bm = adj[b];
    A.erase(b);
    Bm.erase(a);
    for (const auto& kv : Bm) {
      const uint32_t d = kv.first;
      auto it = A.find(d);
      const double s = (it != A.end() ? it->second : 0.0) + kv.second;
      A[d] = s;
      auto& D = adj[d];
      D.erase(b);
      D[a] = s;
    }
    std::unordered_map<uint32_t, double>().swap(Bm);
  }
};

// smallest position > x holding a value <= t (sizes of alive clusters; dead = inf)
struct MinTree {
  uint64_t n = 1;
  std::vector<uint64_t> t;
  explicit MinTree(uint64_t m) {
    while (n < m) n <<= 1;
    t.assign(2 * n, std::numeric_limits<uint64_t>::max());
  }
  void set(uint64_t i, uint64_t v) {
    i += n;
    t[i] = v;
    for (i >>= 1; i; i >>= 1) t[i] = std::min(t[2 * i], t[2 * i + 1]);
  }
  int64_t first_after(uint64_t x, uint64_t limit) const {  // smallest i > x with t[i] <= limit
    return find(1, 0, n, x + 1, limit);
  }
  int64_t find(uint64_t node, uint64_t lo, uint64_t hi, uint64_t from, uint64_t limit) const {
    if (hi <= from || t[node] > limit) return -1;
    if (hi - lo == 1) return (int64_t)lo;
    const uint64_t mid = (lo + hi) / 2;
    const int64_t l = find(2 * node, lo, mid, from, limit);
    return l >= 0 ? l : find(2 * node + 1, mid, hi, from, limit);
  }
};

thread_local std::string g_flt_error;

}  // namespace

extern "C" {

int gomix_fos_bounded_flt(uint64_t num_vertices, uint64_t num_edges, const uint32_t* edge_u,
                          const uint32_t* edge_v, const double* edge_w, uint64_t bound, int32_t weighted,
                          uint64_t* num_sets, uint64_t* total_vars, uint64_t* set_offset, uint32_t* set_vars) {
  try {
    const uint64_t n = num_vertices;
    if (n < 2) throw std::invalid_argument("linkage: need at least two variables");
    if (num_edges && (!edge_u || !edge_v || (weighted && !edge_w)))
      throw std::invalid_argument("linkage: missing edge arrays");
    Flt F;
    F.n = n;
    F.bound = bound == 0 ? n : bound;  // 0: unbounded FLT
    F.alive.assign(n, 1);
    F.size.assign(n, 1);
    F.version.assign(n, 0);
    F.members.resize(n);
    F.adj.resize(n);
    F.remaining = n;
    for (uint64_t v = 0; v < n; ++v) F.members[v] = {(uint32_t)v};
    for (uint64_t i = 0; i < num_edges; ++i) {
      const uint32_t a = edge_u[i], b = edge_v[i];
      if (a >= n || b >= n || a == b) throw std::invalid_argument("maxcut: bad edge");
      const double s = weighted ? std::fabs(edge_w[i]) : 1.0;
      F.adj[a][b] = s;  // SimilarityMatrix::set overwrites: last edge wins (edges are unique)
      F.adj[b][a] = s;
    }
    // ---- phase 1: positive-score merges ------------------------------------
    std::priority_queue<Cand, std::vector<Cand>, HeapOrder> heap;
    auto push = [&](uint32_t a, uint32_t d, double s) {
      if (!(s > 0.0) || F.size[a] + F.size[d] > F.bound) return;
      const uint32_t ka = std::min(a, d), kb = std::max(a, d);
      heap.push(Cand{s, (double)F.size[a] * (double)F.size[d], ka, kb, F.version[ka], F.version[kb]});
    };
    for (uint32_t a = 0; a < n; ++a)
      for (const auto& kv : F.adj[a])
        if (a < kv.first) push(a, kv.first, kv.second);
    while (F.remaining > 1 && !heap.empty()) {
      const Cand c = heap.top();
      heap.pop();
      if (!F.alive[c.ka] || !F.alive[c.kb] || F.version[c.ka] != c.va || F.version[c.kb] != c.vb) continue;
      F.merge(c.ka, c.kb);
      for (const auto& kv : F.adj[c.ka]) push(c.ka, kv.first, kv.second);
    }
    // ---- phase 2: score-0 merges, lexicographic in representatives -----------
    if (F.remaining > 1) {
      MinTree T(n);
      for (uint64_t v = 0; v < n; ++v)
        if (F.alive[v]) T.set(v, F.size[v]);
      uint64_t x = 0;
      while (F.remaining > 1 && x < n) {
        if (!F.alive[x] || F.size[x] >= F.bound) {
          ++x;
          continue;
        }
        const int64_t y = T.first_after(x, F.bound - F.size[x]);
        if (y < 0) {  // x can never merge again: every other cluster only grows
          ++x;
          continue;
        }
        F.merge((uint32_t)x, (uint32_t)y);
        T.set((uint64_t)y, std::numeric_limits<uint64_t>::max());
        T.set(x, F.size[x]);
      }
    }
    // ---- output: singletons, then merged sets in merge order -----------------
    uint64_t total = n;
    for (const auto& s : F.sets) total += s.size();
    if (num_sets) *num_sets = n + F.sets.size();
    if (total_vars) *total_vars = total;
    if (set_offset && set_vars) {
      uint64_t at = 0, k = 0;
      set_offset[0] = 0;
      for (uint64_t v = 0; v < n; ++v) {
        set_vars[at++] = (uint32_t)v;
        set_offset[++k] = at;
      }
      for (const auto& s : F.sets) {
        for (uint32_t v : s) set_vars[at++] = v;
        set_offset[++k] = at;
      }
    }
    return GOMIX_OK;
  } catch (const std::invalid_argument& e) {
    g_flt_error = e.what();
    return GOMIX_E_INVALID;
  } catch (const std::exception& e) {
    g_flt_error = e.what();
    return GOMIX_E_OOM;
  }
}

}  // extern "C"
