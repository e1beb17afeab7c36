// Elimination-order passes over the line graph (host, C++).
//
// Restates, for speed, the reference's ordering passes
//   _eliminate       /root/reference/pkg/src/qtnsim/ordering.py:79-90
//   _run_pass        ordering.py:106-124
//   _choose_min_degree ordering.py:127-129
//   _boltzmann_chooser ordering.py:139-151
//   rgreedy_order    ordering.py:154-189
// with results identical to the reference: the random variates and the
// Boltzmann weight table exp(-d/temp) are produced by numpy on the Python side
// (paper_2106_15740_b200/ordering.py) exactly as the reference draws them, and
// the cumulative-sum / searchsorted selection below repeats the reference's
// float64 arithmetic in the same order.  Adjacency is a bitset per vertex, so
// eliminating v costs deg(v) * nv/64 word operations.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "qtn_internal.h"

namespace {

struct Graph {
  int nv = 0, words = 0;
  std::vector<uint64_t> bits;  // nv x words
  uint64_t* row(int v) { return bits.data() + (size_t)v * words; }
};

bool build_graph(int nv, int n_edges, const int32_t* off, const int32_t* vs, Graph& g) {
  g.nv = nv;
  g.words = (nv + 63) / 64;
  g.bits.assign((size_t)nv * std::max(g.words, 1), 0);
  for (int e = 0; e < n_edges; ++e) {
    for (int a = off[e]; a < off[e + 1]; ++a) {
      int x = vs[a];
      if (x < 0 || x >= nv) return false;
      for (int b = off[e]; b < off[e + 1]; ++b) {
        int y = vs[b];
        if (y < 0 || y >= nv) return false;
        if (x != y) g.row(x)[y >> 6] |= 1ull << (y & 63);
      }
    }
  }
  return true;
}

int popcount_row(const uint64_t* r, int words) {
  int c = 0;
  for (int w = 0; w < words; ++w) c += __builtin_popcountll(r[w]);
  return c;
}

// ordering.py:79-90: neighbours of v become a clique, v disappears.
// Returns the rank of the produced intermediate (= degree of v).
int eliminate(Graph& g, int v, std::vector<int>& nb) {
  nb.clear();
  uint64_t* rv = g.row(v);
  for (int w = 0; w < g.words; ++w) {
    uint64_t m = rv[w];
    while (m) {
      int b = __builtin_ctzll(m);
      nb.push_back(w * 64 + b);
      m &= m - 1;
    }
  }
  for (int a : nb) {
    uint64_t* ra = g.row(a);
    for (int w = 0; w < g.words; ++w) ra[w] |= rv[w];
    ra[a >> 6] &= ~(1ull << (a & 63));
    ra[v >> 6] &= ~(1ull << (v & 63));
  }
  std::memset(rv, 0, sizeof(uint64_t) * g.words);
  return (int)nb.size();
}

constexpr int64_t kDead = std::numeric_limits<int64_t>::max();  // ordering.py:103

// One pass (ordering.py:106-124).  draws == nullptr: min-degree pass.
void run_pass(Graph& g, const double* draws, const double* exp_table, bool temp_zero,
              int32_t* order, int32_t* ranks) {
  const int nv = g.nv;
  std::vector<int64_t> deg(nv);
  for (int v = 0; v < nv; ++v) deg[v] = popcount_row(g.row(v), g.words);
  std::vector<int> nb;
  std::vector<double> cum(nv);
  for (int step = 0; step < nv; ++step) {
    int v = 0;
    if (!draws) {
      // np.argmin: first minimum (ordering.py:127-129)
      int64_t best = deg[0];
      for (int i = 1; i < nv; ++i)
        if (deg[i] < best) { best = deg[i]; v = i; }
    } else {
      int64_t low = kDead;
      for (int i = 0; i < nv; ++i)
        if (deg[i] != kDead && deg[i] < low) low = deg[i];
      // weights then cumsum, sequential float64 adds (ordering.py:143-147)
      double acc = 0.0;
      for (int i = 0; i < nv; ++i) {
        double w = 0.0;
        if (deg[i] != kDead) {
          if (temp_zero)
            w = (deg[i] == low) ? 1.0 : 0.0;
          else
            w = exp_table[deg[i] - low];
        }
        acc += w;
        cum[i] = acc;
      }
      double draw = draws[step] * cum[nv - 1];
      // searchsorted(side="right"): first i with cum[i] > draw
      v = (int)(std::upper_bound(cum.begin(), cum.end(), draw) - cum.begin());
      if (v >= nv) v = nv - 1;  // unreachable for draws in [0, 1)
    }
    ranks[step] = eliminate(g, v, nb);
    for (int a : nb) deg[a] = popcount_row(g.row(a), g.words);
    deg[v] = kDead;
    order[step] = v;
  }
}

double flops_of(const int32_t* ranks, int n) {
  // ordering.py:60-61, summed in step order like the reference
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += std::ldexp(1.0, ranks[i] + 1);
  return s;
}

}  // namespace

extern "C" int qtn_order_pass(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                              const int32_t* edge_vertices, const double* draws,
                              const double* exp_table, int32_t temp_is_zero,
                              int32_t* out_order, int32_t* out_ranks) {
  if (nv < 0 || n_edges < 0 || (draws && !temp_is_zero && !exp_table)) {
    qtn::set_error("qtn_order_pass: bad arguments");
    return QTN_EINVAL;
  }
  Graph g;
  if (!build_graph(nv, n_edges, edge_offsets, edge_vertices, g)) {
    qtn::set_error("hyperedge references unknown vertex");
    return QTN_EINVAL;
  }
  run_pass(g, draws, exp_table, temp_is_zero != 0, out_order, out_ranks);
  return QTN_OK;
}

extern "C" int qtn_rgreedy(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                           const int32_t* edge_vertices, int32_t n_repeats,
                           const double* draws, const double* exp_table,
                           int32_t temp_is_zero, int32_t* out_order, int32_t* out_ranks,
                           int32_t* out_best) {
  if (n_repeats < 1) {
    qtn::set_error("n_repeats must be >= 1");
    return QTN_EINVAL;
  }
  Graph base;
  if (!build_graph(nv, n_edges, edge_offsets, edge_vertices, base)) {
    qtn::set_error("hyperedge references unknown vertex");
    return QTN_EINVAL;
  }
  std::vector<int32_t> order(nv), ranks(nv);
  int best_w = -1, best_rep = -1;
  double best_f = 0.0;
  for (int rep = 0; rep < n_repeats; ++rep) {
    Graph g = base;
    const double* d = rep == 0 ? nullptr : draws + (size_t)(rep - 1) * nv;
    run_pass(g, d, exp_table, temp_is_zero != 0, order.data(), ranks.data());
    int w = 0;
    for (int i = 0; i < nv; ++i) w = std::max(w, (int)ranks[i]);
    double f = flops_of(ranks.data(), nv);
    // key (width, flops_sum, pass), strict less (ordering.py:181-183)
    if (best_rep < 0 || w < best_w || (w == best_w && f < best_f)) {
      best_w = w;
      best_f = f;
      best_rep = rep;
      std::copy(order.begin(), order.end(), out_order);
      std::copy(ranks.begin(), ranks.end(), out_ranks);
    }
  }
  if (out_best) *out_best = best_rep;
  return QTN_OK;
}

extern "C" int qtn_order_ranks(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                               const int32_t* edge_vertices, const int32_t* order,
                               int32_t* out_ranks) {
  Graph g;
  if (!build_graph(nv, n_edges, edge_offsets, edge_vertices, g)) {
    qtn::set_error("hyperedge references unknown vertex");
    return QTN_EINVAL;
  }
  std::vector<char> seen(nv, 0);
  for (int i = 0; i < nv; ++i) {
    if (order[i] < 0 || order[i] >= nv || seen[order[i]]) {
      qtn::set_error("order is not a permutation of the line-graph vertices");
      return QTN_EINVAL;
    }
    seen[order[i]] = 1;
  }
  std::vector<int> nb;
  for (int i = 0; i < nv; ++i) out_ranks[i] = eliminate(g, order[i], nb);
  return QTN_OK;
}
