// run_distributed → DistOutcome on the device path (dist.hpp:138-150,
// dist_common.cpp:117-222): one host thread per rank (SimRuntime::run's
// thread-per-rank model, runtime.cpp:270-285), each owning a Trainer on its
// GPU, then the global results assembled on the host with the reference's
// bitwise replica checks.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "trainer.hpp"

namespace cagnet {

// Where the ranks run: one GPU per rank with NCCL / NVLink peer memory, or
// every rank on one GPU through the in-process world (comm_local.hpp).
enum class Backend : int { Auto = 0, Nccl = 1, Local = 2 };

struct RunOptions {
  bool reassociate = false;
  bool graph = true;
  bool resident_sparse = true;
  bool p2p = true;
  bool overlap = false;
  bool pipeline = false;
  int fuse = 1;
};

// dist.hpp:138-147, fp32 device results widened to fp64.
struct DistOutcome {
  int64_t n = 0;
  std::vector<int64_t> dims;
  std::vector<double> losses;              // per epoch (verified equal on every rank)
  std::vector<double> h_final;             // n x dims.back(), row major
  std::vector<std::vector<double>> y_final;  // layer l: dims[l] x dims[l+1]
  std::vector<std::vector<double>> g_final;  // layer l: n x dims[l+1]
  std::vector<std::vector<double>> weights;  // the verified final model
  double learning_rate = 0;
  // ledger[rank][category] = {messages, words_sent, words_received, payload_words, calls}
  std::vector<std::array<std::array<uint64_t, 5>, kNumCategories>> ledger;
  std::vector<uint64_t> prereduction_totals;  // k-th note summed over ranks (runtime.cpp:287-295)
  std::vector<uint64_t> memory_peaks;         // per rank
  float epoch_ms = 0;                         // last epoch, device time, max over ranks
  int ranks = 0;
  int backend = 0;                            // the backend actually used
};

// Copies a dataset to another GPU (peer copies of the CSR pair, features,
// labels and mask) — per-rank datasets for the NCCL backend.
std::unique_ptr<DeviceDataset> dataset_replicate(const DeviceDataset& d, int device);

DistOutcome run_distributed(const DeviceDataset& data, const std::vector<int64_t>& dims,
                            const double* weights, double lr, const Strategy& strat, int epochs,
                            Backend backend, const RunOptions& opt);

}  // namespace cagnet
