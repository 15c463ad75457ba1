// instances.cu — host-side synthetic Max-Cut instance generators of the
// product library (inputs to the hot path, no device work).
//
//   gomix_generate_torus   : generate_torus (maxcut.hpp:87-147) — same stream,
//                            same draw order, so instances equal the reference's.
//   gomix_generate_regular : random d-regular graph (the reference has none,
//                            SURVEY.md §8(d) C4): configuration-model pairing
//                            from the RngStream, loops / multi-edges removed by
//                            random double-edge swaps; weights unit, uniform_int
//                            or uniform_real (rng.hpp:38-43).
#include <algorithm>
#include <cstring>
#include <unordered_set>
#include <vector>

#include "gomix_gpu.h"
#include "internal.cuh"

using namespace gomix_b200;

namespace {

struct Edge {
  uint32_t u, v;
  double w;
};

double draw_weight(ReplayStream& rng, int kind, int64_t lo, int64_t hi) {
  if (kind == 0) return 1.0;
  if (kind == 1) return (double)(lo + (int64_t)rng.uniform_index((uint64_t)(hi - lo) + 1));
  return (double)(rng.next() >> 11) * 0x1.0p-53;  // uniform_real (rng.hpp:43)
}

void emit(std::vector<Edge>& e, uint32_t* eu, uint32_t* ev, double* ew) {
  std::sort(e.begin(), e.end(), [](const Edge& a, const Edge& b) {
    return a.u != b.u ? a.u < b.u : a.v < b.v;
  });
  for (size_t i = 0; i < e.size(); ++i) {
    eu[i] = e[i].u;
    ev[i] = e[i].v;
    ew[i] = e[i].w;
  }
}

thread_local std::string g_gen_error;

}  // namespace

extern "C" {

int gomix_generate_torus(uint64_t width, uint64_t height, int32_t weight_kind, int64_t lo,
                         int64_t hi, uint64_t seed, uint32_t* eu, uint32_t* ev, double* ew) {
  if (width < 3 || height < 3 || !eu || !ev || !ew) return GOMIX_E_INVALID;
  if (weight_kind == 1 && lo > hi) return GOMIX_E_INVALID;
  if (width * height >= (1ull << 31)) return GOMIX_E_INVALID;
  ReplayStream rng(seed);
  std::vector<Edge> e;
  e.reserve(2 * width * height);
  for (uint64_t r = 0; r < height; ++r)
    for (uint64_t c = 0; c < width; ++c) {
      const uint64_t v = r * width + c;
      const uint64_t nb[2] = {r * width + (c + 1) % width, ((r + 1) % height) * width + c};
      for (uint64_t x : nb) {
        const double w = draw_weight(rng, weight_kind, lo, hi);
        e.push_back({(uint32_t)std::min(v, x), (uint32_t)std::max(v, x), w});
      }
    }
  emit(e, eu, ev, ew);
  return GOMIX_OK;
}

int gomix_generate_regular(uint64_t num_vertices, uint32_t degree, int32_t weight_kind, int64_t lo,
                           int64_t hi, uint64_t seed, uint32_t* eu, uint32_t* ev, double* ew) {
  const uint64_t nv = num_vertices, d = degree;
  if (nv < 2 || d == 0 || d >= nv || (nv * d) % 2 || !eu || !ev || !ew) return GOMIX_E_INVALID;
  if (weight_kind == 1 && lo > hi) return GOMIX_E_INVALID;
  ReplayStream rng(seed);
  const uint64_t q = nv * d / 2;
  std::vector<uint32_t> stubs(nv * d);
  for (uint64_t i = 0; i < nv * d; ++i) stubs[i] = (uint32_t)(i / d);
  for (uint64_t i = stubs.size(); i > 1; --i) std::swap(stubs[i - 1], stubs[rng.uniform_index(i)]);
  std::vector<std::pair<uint32_t, uint32_t>> pr(q);
  auto key = [nv](uint32_t a, uint32_t b) {
    return a < b ? (uint64_t)a * nv + b : (uint64_t)b * nv + a;
  };
  std::unordered_multiset<uint64_t> seen;
  seen.reserve(q * 2);
  for (uint64_t i = 0; i < q; ++i) {
    pr[i] = {stubs[2 * i], stubs[2 * i + 1]};
    seen.insert(key(pr[i].first, pr[i].second));
  }
  auto bad = [&](uint64_t i) {
    return pr[i].first == pr[i].second || seen.count(key(pr[i].first, pr[i].second)) > 1;
  };
  // random double-edge swaps until simple: (a,b),(c,e) -> (a,c),(b,e)
  for (uint64_t sweep = 0; sweep < 1000; ++sweep) {
    bool any = false;
    for (uint64_t i = 0; i < q; ++i) {
      if (!bad(i)) continue;
      any = true;
      const uint64_t j = rng.uniform_index(q);
      if (j == i) continue;
      const uint32_t a = pr[i].first, b = pr[i].second, c = pr[j].first, x = pr[j].second;
      if (a == c || b == x || seen.count(key(a, c)) || seen.count(key(b, x))) continue;
      seen.erase(seen.find(key(a, b)));
      seen.erase(seen.find(key(c, x)));
      pr[i] = {a, c};
      pr[j] = {b, x};
      seen.insert(key(a, c));
      seen.insert(key(b, x));
    }
    if (!any) break;
    if (sweep == 999) return GOMIX_E_STATE;
  }
  std::sort(pr.begin(), pr.end(), [](auto& l, auto& r) {
    const uint32_t lu = std::min(l.first, l.second), ru = std::min(r.first, r.second);
    const uint32_t lv = std::max(l.first, l.second), rv = std::max(r.first, r.second);
    return lu != ru ? lu < ru : lv < rv;
  });
  std::vector<Edge> e(q);
  for (uint64_t i = 0; i < q; ++i)
    e[i] = {std::min(pr[i].first, pr[i].second), std::max(pr[i].first, pr[i].second),
            draw_weight(rng, weight_kind, lo, hi)};
  emit(e, eu, ev, ew);
  return GOMIX_OK;
}

}  // extern "C"
