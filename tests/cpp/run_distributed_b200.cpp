// TEST — the INTEGRATION.md adapter, compiled: the reference's own C++ types
// (/root/reference/proj/include) driving libcagnet_b200.so through the C-ABI.
//
//   run_distributed_b200(data, raw, model, strat, epochs)  ==  run_distributed (dist.hpp:149-150)
//
// main() builds the reference dataset and model from the harness seeds
// (harness.hpp:35-45), runs the reference's run_distributed (oracle/_ref, the
// unmodified sources) and the adapter on the same inputs, and compares them
// the way verify_against_serial does (harness.cpp:118-166): rel_frobenius
// (dense.cpp:190-201) of h_final and every y / g / w <= 1e-4, per-epoch
// |dloss| / max(1, |loss|) <= 1e-4, and — on the reference's communication
// schedule — the ledger word for word and the 3D prereduction / memory gauges.
// Exit status 0 = every case passed.  Built by tests/cpp/Makefile; run by
// tests/test_cpp_adapter.py on a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "cagnet/dataset.hpp"
#include "cagnet/dist.hpp"
#include "cagnet/gnn.hpp"
#include "cagnet_b200.h"

namespace cagnet {

static void ok(int rc) {
  if (rc != CAGNET_OK) throw std::runtime_error(std::string("cagnet: ") + cagnet_last_error());
}

// The adapter a maintainer adds beside src/dist_common.cpp.  `raw` is the
// unnormalised adjacency `data` was made from (make_dataset normalises on
// the device, bit-exactly like csr.cpp:94-116).
DistOutcome run_distributed_b200(const GraphDataset& data, const CsrMatrix& raw, const GnnModel& model,
                                 const Strategy& strat, int epochs, uint32_t options = 0) {
  const int64_t n = static_cast<int64_t>(data.n);
  std::vector<int64_t> rp(raw.row_ptr.begin(), raw.row_ptr.end());
  std::vector<int64_t> ci(raw.col_idx.begin(), raw.col_idx.end());
  std::vector<int64_t> labels(data.labels.begin(), data.labels.end());
  cagnet_dataset_t g = nullptr;
  ok(cagnet_dataset_make(0, n, rp.data(), ci.data(), data.features.data(),
                         static_cast<int64_t>(data.features.cols()), labels.data(), data.train_mask.data(),
                         static_cast<int64_t>(data.num_classes), &g));
  std::vector<int64_t> dims(model.layer_dims.begin(), model.layer_dims.end());
  std::vector<double> w;
  for (const DenseMatrix& W : model.weights) w.insert(w.end(), W.data(), W.data() + W.words());
  cagnet_outcome_t o = nullptr;
  const int rc = cagnet_run_distributed(g, dims.data(), static_cast<int>(dims.size()), w.data(),
                                        model.learning_rate, static_cast<int>(strat.kind), strat.ranks,
                                        strat.repl, static_cast<int>(strat.block), epochs,
                                        CAGNET_BACKEND_AUTO, options, &o);
  cagnet_dataset_free(g);
  ok(rc);
  int64_t info[8];
  ok(cagnet_outcome_info(o, info));
  DistOutcome out;
  out.losses.resize(static_cast<size_t>(info[2]));
  ok(cagnet_outcome_losses(o, out.losses.data()));
  out.h_final = DenseMatrix(data.n, model.layer_dims.back());
  ok(cagnet_outcome_h_final(o, out.h_final.data()));
  out.model = model;
  for (size_t l = 0; l + 1 < model.layer_dims.size(); ++l) {
    DenseMatrix y(model.layer_dims[l], model.layer_dims[l + 1]);
    ok(cagnet_outcome_y(o, static_cast<int>(l), y.data()));
    out.y_final.push_back(std::move(y));
    DenseMatrix gg(data.n, model.layer_dims[l + 1]);
    ok(cagnet_outcome_g(o, static_cast<int>(l), gg.data()));
    out.g_final.push_back(std::move(gg));
    ok(cagnet_outcome_weight(o, static_cast<int>(l), out.model.weights[l].data()));
  }
  out.ledger = CommLedger(strat.ranks);
  for (int r = 0; r < strat.ranks; ++r) {
    uint64_t led[20];
    ok(cagnet_outcome_ledger(o, r, led));
    for (int c = 0; c < 4; ++c) {
      CommCounter& k = out.ledger.at(static_cast<Category>(c), r);
      k.messages = led[5 * c];
      k.words_sent = led[5 * c + 1];
      k.words_received = led[5 * c + 2];
      k.payload_words = led[5 * c + 3];
      k.calls = led[5 * c + 4];
    }
  }
  out.prereduction_totals.resize(static_cast<size_t>(info[5]));
  if (info[5]) ok(cagnet_outcome_prereduction_totals(o, out.prereduction_totals.data()));
  out.memory_peaks.resize(static_cast<size_t>(strat.ranks));
  ok(cagnet_outcome_memory_peaks(o, out.memory_peaks.data()));
  ok(cagnet_outcome_free(o));
  return out;
}

}  // namespace cagnet

using namespace cagnet;

struct Case {
  const char* name;
  StrategyKind kind;
  int ranks, repl, block;
  std::size_t n;
  std::vector<std::size_t> dims;
};

int main() {
  const std::vector<Case> cases = {
      {"serial-1d", StrategyKind::OneD, 1, 1, 0, 64, {12, 8, 5}},
      {"1d-p4", StrategyKind::OneD, 4, 1, 0, 70, {12, 8, 5}},
      {"1.5d-p4-c2", StrategyKind::OneFiveD, 4, 2, 0, 70, {12, 8, 6, 5}},
      {"2d-p4-b2", StrategyKind::TwoD, 4, 1, 2, 50, {12, 8, 5}},
      {"3d-p8", StrategyKind::ThreeD, 8, 1, 0, 45, {12, 8, 8, 5}},
  };
  const int epochs = 3;
  int failures = 0;
  for (const Case& c : cases) {
    // harness seeds: graph 1, features 2, labels 3, weights 4 (harness.hpp:35-45)
    const CsrMatrix raw = generate_erdos_renyi(c.n, 6.0, 1);
    const GraphDataset data = make_dataset(raw, random_features(c.n, c.dims.front(), 2),
                                           random_labels(c.n, c.dims.back(), 3),
                                           std::vector<std::uint8_t>(c.n, 1), c.dims.back());
    const GnnModel model = init_glorot(c.dims, 4, 0.5);
    Strategy s;
    s.kind = c.kind;
    s.ranks = c.ranks;
    s.repl = c.repl;
    s.block = static_cast<std::size_t>(c.block);
    const DistOutcome want = run_distributed(data, model, s, epochs, Scheduler::Concurrent);
    // The reference's communication schedule (per-stage sparse broadcasts,
    // reference propagation order) so the ledgers must match word for word.
    const DistOutcome got = run_distributed_b200(data, raw, model, s, epochs, CAGNET_OPT_NO_RESIDENT_SPARSE);
    double worst = 0;
    for (size_t e = 0; e < want.losses.size(); ++e)
      worst = std::max(worst, std::fabs(got.losses[e] - want.losses[e]) / std::max(1.0, std::fabs(want.losses[e])));
    worst = std::max(worst, rel_frobenius(got.h_final, want.h_final));
    for (size_t l = 0; l < want.y_final.size(); ++l) {
      worst = std::max(worst, rel_frobenius(got.y_final[l], want.y_final[l]));
      worst = std::max(worst, rel_frobenius(got.g_final[l], want.g_final[l]));
      worst = std::max(worst, rel_frobenius(got.model.weights[l], want.model.weights[l]));
    }
    bool ledger_ok = true;
    for (int cat = 0; cat < 4; ++cat)
      for (int r = 0; r < s.ranks; ++r) {
        const CommCounter& a = got.ledger.at(static_cast<Category>(cat), r);
        const CommCounter& b = want.ledger.at(static_cast<Category>(cat), r);
        ledger_ok = ledger_ok && a.messages == b.messages && a.words_sent == b.words_sent &&
                    a.words_received == b.words_received && a.payload_words == b.payload_words &&
                    a.calls == b.calls;
      }
    const bool gauges_ok = got.prereduction_totals == want.prereduction_totals && got.memory_peaks == want.memory_peaks;
    const bool pass = worst <= 1e-4 && ledger_ok && gauges_ok;
    std::printf("%-12s ranks=%d  max_rel=%.3e  ledger=%s  gauges=%s (%zu prereductions)  %s\n", c.name, s.ranks,
                worst, ledger_ok ? "equal" : "DIFFERENT", gauges_ok ? "equal" : "DIFFERENT",
                want.prereduction_totals.size(), pass ? "PASS" : "FAIL");
    failures += pass ? 0 : 1;
  }
  return failures == 0 ? 0 : 1;
}
