// run_distributed → DistOutcome (see run.hpp).
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "run.hpp"

namespace cagnet {

namespace {

DeviceCsr csr_to_device(const DeviceCsr& a, int device, cudaStream_t s) {
  DeviceCsr o;
  o.device = device;
  o.n_rows = a.n_rows;
  o.n_cols = a.n_cols;
  o.nnz = a.nnz;
  o.row_ptr.resize(static_cast<size_t>(a.n_rows + 1));
  o.col_idx.resize(static_cast<size_t>(a.nnz > 0 ? a.nnz : 1));
  o.vals.resize(static_cast<size_t>(a.nnz > 0 ? a.nnz : 1));
  CG_CUDA(cudaMemcpyPeerAsync(o.row_ptr.get(), device, a.row_ptr.get(), a.device, (a.n_rows + 1) * sizeof(int64_t), s));
  if (a.nnz) {
    CG_CUDA(cudaMemcpyPeerAsync(o.col_idx.get(), device, a.col_idx.get(), a.device, a.nnz * sizeof(int32_t), s));
    CG_CUDA(cudaMemcpyPeerAsync(o.vals.get(), device, a.vals.get(), a.device, a.nnz * sizeof(float), s));
  }
  return o;
}

// Host copy of one rank's tile, dense rows x cols.
struct HostTile {
  int64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  int owner = 0;
  std::vector<float> v;
};

// Trainer::assemble_tiles (dist_common.cpp:117-145): each tile lands at its
// (rows, cols) range; a replicated tile must equal its owner's bit for bit.
std::vector<double> assemble(int64_t n, int64_t width, const std::vector<HostTile>& tiles) {
  std::vector<double> out(static_cast<size_t>(n * width), 0.0);
  for (size_t r = 0; r < tiles.size(); ++r) {
    const HostTile& t = tiles[r];
    const int64_t rows = t.r1 - t.r0, cols = t.c1 - t.c0;
    if (static_cast<int64_t>(t.v.size()) != rows * cols)
      throw std::logic_error("assemble: rank " + std::to_string(r) + " tile has " + std::to_string(t.v.size()) +
                             " values, expected " + std::to_string(rows) + "x" + std::to_string(cols));
    if (t.owner != static_cast<int>(r)) {
      const HostTile& o = tiles[static_cast<size_t>(t.owner)];
      if (o.v.size() != t.v.size() || std::memcmp(o.v.data(), t.v.data(), t.v.size() * sizeof(float)) != 0)
        throw std::runtime_error("replica divergence: rank " + std::to_string(r) + " disagrees with rank " +
                                 std::to_string(t.owner));
      continue;
    }
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols; ++j)
        out[static_cast<size_t>((t.r0 + i) * width + t.c0 + j)] = t.v[static_cast<size_t>(i * cols + j)];
  }
  return out;
}

std::vector<double> widen(const std::vector<float>& v) { return std::vector<double>(v.begin(), v.end()); }

}  // namespace

std::unique_ptr<DeviceDataset> dataset_replicate(const DeviceDataset& d, int device) {
  CG_CUDA(cudaSetDevice(device));
  auto o = std::make_unique<DeviceDataset>();
  o->device = device;
  o->n = d.n;
  o->f = d.f;
  o->num_classes = d.num_classes;
  o->train_count = d.train_count;
  o->ldf = d.ldf;
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    o->adj = csr_to_device(d.adj, device, s);
    o->adj_t = csr_to_device(d.adj_t, device, s);
    o->features.resize(static_cast<size_t>(d.n * d.ldf > 0 ? d.n * d.ldf : 1));
    o->labels.resize(static_cast<size_t>(d.n > 0 ? d.n : 1));
    o->mask.resize(static_cast<size_t>(d.n > 0 ? d.n : 1));
    if (d.n) {
      CG_CUDA(cudaMemcpyPeerAsync(o->features.get(), device, d.features.get(), d.device,
                                  d.n * d.ldf * sizeof(float), s));
      CG_CUDA(cudaMemcpyPeerAsync(o->labels.get(), device, d.labels.get(), d.device, d.n * sizeof(int32_t), s));
      CG_CUDA(cudaMemcpyPeerAsync(o->mask.get(), device, d.mask.get(), d.device, d.n, s));
    }
    CG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  return o;
}

DistOutcome run_distributed(const DeviceDataset& data, const std::vector<int64_t>& dims,
                            const double* weights, double lr, const Strategy& strat, int epochs,
                            Backend backend, const RunOptions& opt) {
  if (epochs <= 0) throw std::invalid_argument("run_epochs: epoch count must be positive");
  const ProcessGrid grid = ProcessGrid::make(strat);  // validates before any GPU work
  const int P = grid.ranks();
  int n_dev = 0;
  CG_CUDA(cudaGetDeviceCount(&n_dev));
  if (backend == Backend::Auto) backend = (P > 1 && n_dev < P) ? Backend::Local : Backend::Nccl;
  if (backend == Backend::Nccl && P > 1 && n_dev < P)
    throw std::invalid_argument("run_distributed: " + std::to_string(P) + " ranks need " + std::to_string(P) +
                                " GPUs for the NCCL backend, found " + std::to_string(n_dev));

  // Communicator id and the per-rank datasets.
  std::vector<uint8_t> id(128, 0);
  std::vector<int> device(static_cast<size_t>(P), data.device);
  std::vector<std::unique_ptr<DeviceDataset>> copies(static_cast<size_t>(P));
  if (P > 1) {
    if (backend == Backend::Local) {
      LocalId lid;
      LocalWorld::create(P, data.device, &lid);
      std::memcpy(id.data(), &lid, sizeof(lid));
    } else {
      ncclUniqueId nid;
      CG_NCCL(ncclGetUniqueId(&nid));
      std::memcpy(id.data(), &nid, sizeof(nid));
      for (int r = 0; r < P; ++r) {
        device[static_cast<size_t>(r)] = r;
        if (r != data.device) copies[static_cast<size_t>(r)] = dataset_replicate(data, r);
      }
    }
  }

  std::vector<std::unique_ptr<Trainer>> trainers(static_cast<size_t>(P));
  std::vector<std::vector<double>> losses(static_cast<size_t>(P));
  std::vector<std::exception_ptr> errors(static_cast<size_t>(P));
  std::mutex mu;
  auto body = [&](int r) {
    try {
      CG_CUDA(cudaSetDevice(device[static_cast<size_t>(r)]));
      const DeviceDataset& mine = copies[static_cast<size_t>(r)] ? *copies[static_cast<size_t>(r)] : data;
      auto t = make_trainer(mine, dims, weights, lr, strat, r,
                            P > 1 ? reinterpret_cast<const ncclUniqueId*>(id.data()) : nullptr);
      t->set_graph(opt.graph);
      t->set_reassociate(opt.reassociate);
      t->set_fuse(opt.fuse);
      t->set_resident_sparse(opt.resident_sparse);
      t->set_p2p(opt.p2p);
      t->set_overlap(opt.overlap);
      t->set_pipeline(opt.pipeline);
      t->distribute();
      losses[static_cast<size_t>(r)] = t->run_epochs(epochs);
      trainers[static_cast<size_t>(r)] = std::move(t);
    } catch (...) {
      errors[static_cast<size_t>(r)] = std::current_exception();
      if (backend == Backend::Local && P > 1) {
        // Release the peers blocked in this rank's collectives.
        LocalId lid;
        std::memcpy(&lid, id.data(), sizeof(lid));
        std::string why = "rank " + std::to_string(r) + " failed";
        try {
          std::rethrow_exception(errors[static_cast<size_t>(r)]);
        } catch (const std::exception& e) {
          why += ": " + std::string(e.what());
        } catch (...) {
        }
        std::lock_guard<std::mutex> lk(mu);
        LocalWorld::abort_id(lid, why);
      }
    }
  };
  if (P == 1) {
    body(0);
  } else {
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r) th.emplace_back(body, r);
    for (auto& x : th) x.join();
  }
  // The lowest-rank original failure wins (runtime.cpp:281-284); peers
  // released by an abort only echo it.
  std::exception_ptr first, echo;
  for (int r = 0; r < P; ++r) {
    if (!errors[static_cast<size_t>(r)]) continue;
    bool is_echo = false;
    try {
      std::rethrow_exception(errors[static_cast<size_t>(r)]);
    } catch (const std::exception& e) {
      is_echo = std::string(e.what()).find("local world aborted") != std::string::npos;
    } catch (...) {
    }
    if (!is_echo && !first) first = errors[static_cast<size_t>(r)];
    if (is_echo && !echo) echo = errors[static_cast<size_t>(r)];
  }
  if (first) std::rethrow_exception(first);
  if (echo) std::rethrow_exception(echo);

  DistOutcome out;
  out.n = data.n;
  out.dims = dims;
  out.ranks = P;
  out.backend = static_cast<int>(backend);
  out.learning_rate = lr;
  const int L = static_cast<int>(dims.size());
  // verified_losses (dist_common.cpp:181-192)
  for (int r = 1; r < P; ++r)
    if (losses[static_cast<size_t>(r)].size() != losses[0].size() ||
        (!losses[0].empty() && std::memcmp(losses[static_cast<size_t>(r)].data(), losses[0].data(),
                                           losses[0].size() * sizeof(double)) != 0))
      throw std::runtime_error("loss replica divergence at rank " + std::to_string(r));
  out.losses = losses[0];
  auto tiles_of = [&](int64_t width, auto&& pick) {
    std::vector<HostTile> tiles(static_cast<size_t>(P));
    for (int r = 0; r < P; ++r) {
      Trainer& t = *trainers[static_cast<size_t>(r)];
      CG_CUDA(cudaSetDevice(t.device()));
      t.sync();
      HostTile& h = tiles[static_cast<size_t>(r)];
      const BlockRange rr = t.tile_rows(r), cc = t.tile_cols(r, width);
      h.r0 = rr.begin;
      h.r1 = rr.end;
      h.c0 = cc.begin;
      h.c1 = cc.end;
      h.owner = t.tile_owner(r);
      h.v.resize(static_cast<size_t>(rr.size() * cc.size()));
      pick(t, h.v.data());
    }
    return tiles;
  };
  out.h_final = assemble(data.n, dims.back(), tiles_of(dims.back(), [&](Trainer& t, float* o) { t.h_tile(L - 1, o); }));
  for (int l = 0; l + 1 < L; ++l)
    out.g_final.push_back(assemble(data.n, dims[static_cast<size_t>(l + 1)],
                                   tiles_of(dims[static_cast<size_t>(l + 1)],
                                            [&](Trainer& t, float* o) { t.g_tile(l, o); })));
  // verified_y / verified_model (dist_common.cpp:152-179): bitwise equal on every rank.
  auto verified = [&](int l, bool y, const char* what) {
    const int64_t cnt = dims[static_cast<size_t>(l)] * dims[static_cast<size_t>(l + 1)];
    std::vector<float> ref(static_cast<size_t>(cnt)), cur(static_cast<size_t>(cnt));
    for (int r = 0; r < P; ++r) {
      Trainer& t = *trainers[static_cast<size_t>(r)];
      CG_CUDA(cudaSetDevice(t.device()));
      float* dst = r == 0 ? ref.data() : cur.data();
      if (y)
        t.ygrad(l, dst);
      else
        t.weight(l, dst);
      if (r > 0 && std::memcmp(ref.data(), cur.data(), ref.size() * sizeof(float)) != 0)
        throw std::runtime_error(std::string(what) + " replica divergence at rank " + std::to_string(r) +
                                 ", layer " + std::to_string(l + 1));
    }
    return widen(ref);
  };
  for (int l = 0; l + 1 < L; ++l) {
    out.y_final.push_back(verified(l, true, "gradient"));
    out.weights.push_back(verified(l, false, "weight"));
  }
  out.ledger.resize(static_cast<size_t>(P));
  out.memory_peaks.assign(static_cast<size_t>(P), 0);
  for (int r = 0; r < P; ++r) {
    Trainer& t = *trainers[static_cast<size_t>(r)];
    for (int c = 0; c < kNumCategories; ++c) {
      const CommCounter& k = t.comm().counter(static_cast<Category>(c));
      out.ledger[static_cast<size_t>(r)][static_cast<size_t>(c)] = {k.messages, k.words_sent, k.words_received,
                                                                     k.payload_words, k.calls};
    }
    const std::vector<uint64_t>& pr = t.prereductions();
    if (pr.size() > out.prereduction_totals.size()) out.prereduction_totals.resize(pr.size(), 0);
    for (size_t i = 0; i < pr.size(); ++i) out.prereduction_totals[i] += pr[i];
    out.memory_peaks[static_cast<size_t>(r)] = t.memory_peak();
    out.epoch_ms = std::max(out.epoch_ms, t.last_epoch_ms());
  }
  // Trainers go before the communication world and the dataset copies.
  for (auto& t : trainers) {
    if (t) CG_CUDA(cudaSetDevice(t->device()));
    t.reset();
  }
  return out;
}

}  // namespace cagnet
