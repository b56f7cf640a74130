// The paper's analytic communication model and its reconciliation with a
// metered ledger (cost.hpp:27-115, cost.cpp:48-161 of the reference), so a
// B200 run's NCCL / peer-memory traffic — metered with the reference's ledger
// conventions (comm.cu) — is checked against the closed forms it should obey:
//   1D   words = L (2nf + f^2)                     messages = L (lg P + 2P)
//   1.5D words = L (2nf/c + 2nfc/P)                messages = L (2P/c^2 + 2 lg c + lg P)
//   2D   words = L (8nf/√P + 2nnz/√P + f^2)        messages = L (4√P + 2 lg P)
//   3D   words = L (2nnz/P^(2/3) + 12nf/P^(2/3))   messages = 4 L ∛P
// (per rank per epoch, integer arithmetic in the order of the formulas;
// lg = ceil(log2)).  1D / 1.5D reconcile exactly, up to the one-word loss
// all-reduce (and 1.5D's replicated weight-gradient all-reduce); 2D / 3D
// within a [0.5, 2] envelope; one rank meters nothing (degenerate).
#pragma once

#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "grid.hpp"

namespace cagnet {
namespace cost {

struct Params {
  int64_t n = 0, nnz = 0, f = 0, layers = 0, ranks = 1, repl = 1;
};

struct Prediction {
  int64_t words = 0, messages = 0;
  std::vector<std::pair<std::string, int64_t>> terms;  // sum to `words`
};

inline int64_t ceil_lg(int64_t p) {
  if (p <= 0) throw std::invalid_argument("ceil_lg: positive argument required");
  int64_t k = 0;
  while ((int64_t{1} << k) < p) ++k;
  return k;
}

inline void check(const Params& p) {
  if (p.n <= 0 || p.f <= 0 || p.layers <= 0 || p.ranks <= 0 || p.repl <= 0 || p.nnz < 0)
    throw std::invalid_argument("cost model: all parameters must be positive");
}

inline Prediction make(std::vector<std::pair<std::string, int64_t>> terms, int64_t messages) {
  Prediction out;
  for (const auto& t : terms) out.words += t.second;
  out.terms = std::move(terms);
  out.messages = messages;
  return out;
}

inline Prediction predict(StrategyKind kind, const Params& p) {
  check(p);
  const int64_t L = p.layers, nf = p.n * p.f, P = p.ranks;
  switch (kind) {
    case StrategyKind::OneD:
      return make({{"embedding_broadcast", L * 2 * nf}, {"weight_gradient_reduce", L * p.f * p.f}},
                  L * (ceil_lg(P) + 2 * P));
    case StrategyKind::OneFiveD: {
      const int64_t c = p.repl;
      if (P % c != 0) throw std::invalid_argument("predict_15d: repl must divide ranks");
      return make({{"embedding_broadcast", L * 2 * nf / c}, {"partial_reduce", L * 2 * nf * c / P}},
                  L * (2 * P / (c * c) + 2 * ceil_lg(c) + ceil_lg(P)));
    }
    case StrategyKind::TwoD: {
      const int64_t s = exact_isqrt(static_cast<int>(P), "predict_2d");
      return make({{"dense_panels", L * 8 * nf / s},
                   {"sparse_panels", L * 2 * p.nnz / s},
                   {"weight_gradient_gather", L * p.f * p.f}},
                  L * (4 * s + 2 * ceil_lg(P)));
    }
    case StrategyKind::ThreeD: {
      const int64_t s = exact_icbrt(static_cast<int>(P), "predict_3d");
      return make({{"sparse_panels", L * 2 * p.nnz / (s * s)}, {"dense_panels", L * 12 * nf / (s * s)}},
                  L * 4 * s);
    }
  }
  throw std::invalid_argument("strategy: unknown kind");
}

// Alpha-beta time of one forward propagation on a rows x cols tile grid.
inline double rect_layer(const Params& p, int64_t rows, int64_t cols, double alpha, double beta) {
  check(p);
  if (rows <= 0 || cols <= 0) throw std::invalid_argument("predict_2d_rect_layer: grid sides must be positive");
  const double nf = static_cast<double>(p.n) * static_cast<double>(p.f);
  const double nnz = static_cast<double>(p.nnz);
  return alpha * static_cast<double>(std::gcd(rows, cols)) +
         beta * (nnz / static_cast<double>(rows) + nf / static_cast<double>(cols) + nf / static_cast<double>(rows));
}

// Aggregate storage in words: serial, 1.5D with the adjacency per layer,
// 1.5D with one adjacency, 3D peak.
struct Footprints {
  int64_t serial = 0, repl15d = 0, repl15d_single_adj = 0, split3d_peak = 0;
};
inline Footprints footprints(int64_t n, int64_t nnz, int64_t f, int64_t fmax, int64_t dims, int64_t repl,
                             int64_t ranks) {
  if (n <= 0 || f <= 0 || fmax <= 0 || dims < 2 || repl <= 0 || ranks <= 0 || nnz < 0)
    throw std::invalid_argument("memory_footprints: bad parameters");
  const int64_t side = exact_icbrt(static_cast<int>(ranks), "memory_footprints");
  return Footprints{nnz + n * f * dims, dims * repl * (nnz + n * f), repl * nnz + dims * repl * n * f,
                    nnz + n * f * (dims - 1) + side * n * fmax};
}

struct Comparison {
  int64_t predicted_words = 0, extra_words = 0;
  double measured_words = 0, ratio = 0;
  bool exact = false, degenerate = false, within_band = false;
};

// payload_words summed over every rank and category, per rank per epoch,
// against the prediction (+ the documented out-of-model words).
inline Comparison compare(StrategyKind kind, const Params& p, uint64_t total_payload_words, int ranks_in_ledger,
                          int epochs) {
  if (epochs <= 0) throw std::invalid_argument("compare_cost: positive epochs required");
  if (ranks_in_ledger != p.ranks)
    throw std::invalid_argument("compare_cost: ledger has " + std::to_string(ranks_in_ledger) +
                                " ranks, parameters say " + std::to_string(p.ranks));
  Comparison c;
  c.predicted_words = predict(kind, p).words;
  if (kind == StrategyKind::OneD) {
    c.extra_words = 1;  // the loss all-reduce
    c.exact = true;
  } else if (kind == StrategyKind::OneFiveD) {
    c.extra_words = p.layers * p.f * p.f + 1;  // replicated Y all-reduce + the loss
    c.exact = true;
  }
  c.measured_words = static_cast<double>(total_payload_words) / (static_cast<double>(p.ranks) * epochs);
  if (p.ranks == 1) {
    c.degenerate = true;
    c.within_band = true;
    return c;
  }
  const double expected = static_cast<double>(c.predicted_words + c.extra_words);
  c.ratio = c.measured_words / expected;
  c.within_band = c.exact ? c.measured_words == expected : (c.ratio >= 0.5 && c.ratio <= 2.0);
  return c;
}

}  // namespace cost
}  // namespace cagnet
