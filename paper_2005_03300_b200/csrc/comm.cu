#include <cstring>

#include "comm.hpp"

#include "nvtx.hpp"

namespace cagnet {

namespace {
size_t dtype_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt8: case ncclUint8: return 1;
    default: return 2;
  }
}
int local_dtype(ncclDataType_t t) {
  if (t == ncclFloat32) return 0;
  if (t == ncclFloat64) return 1;
  throw std::invalid_argument("local collectives: reductions support f32 and f64 only");
}
}  // namespace

Comm::Comm(const ProcessGrid& grid, int rank, const ncclUniqueId* id)
    : rank_(rank), ranks_(grid.ranks()) {
  if (ranks_ == 1) return;
  if (!id) throw std::invalid_argument("Comm: an NCCL unique id is required for P > 1");
  if (is_local_id(id)) {
    LocalId lid;
    std::memcpy(&lid, id, sizeof(lid));
    if (lid.ranks != ranks_)
      throw std::invalid_argument("Comm: local world has " + std::to_string(lid.ranks) + " ranks, grid has " +
                                  std::to_string(ranks_));
    int dev = 0;
    CG_CUDA(cudaGetDevice(&dev));
    if (dev != lid.device)
      throw std::invalid_argument("Comm: local world lives on device " + std::to_string(lid.device) +
                                  " but this rank runs on device " + std::to_string(dev));
    auto w = LocalWorld::attach(lid, rank);
    // Register every group now: flag arenas are allocated outside any capture.
    w->group_flags(grid.world());
    if (grid.kind() != GridKind::Row1D) {
      w->group_flags(grid.row_group(rank));
      w->group_flags(grid.col_group(rank));
    }
    if (grid.has_fiber_groups()) w->group_flags(grid.fiber_group(rank));
    local_ = std::make_unique<LocalCollectives>(std::move(w), rank);
    return;
  }
  CG_NCCL(ncclCommInitRank(&world_, ranks_, *id, rank));
  comms_[grid.world().id] = world_;
  // Split one communicator per group kind, in the same order on every rank.
  auto split = [&](const Group& g) {
    if (comms_.count(g.id)) return;
    ncclComm_t c = nullptr;
    CG_NCCL(ncclCommSplit(world_, g.id, rank, &c, nullptr));
    comms_[g.id] = c;
  };
  if (grid.kind() != GridKind::Row1D) {
    split(grid.row_group(rank));
    split(grid.col_group(rank));
  }
  if (grid.has_fiber_groups()) split(grid.fiber_group(rank));
}

void Comm::check_async() {
  if (local_) {
    local_->world().check();
    return;
  }
  for (auto& kv : comms_) {
    ncclResult_t async = ncclSuccess;
    if (kv.second && ncclCommGetAsyncError(kv.second, &async) == ncclSuccess && async != ncclSuccess &&
        async != ncclInProgress) {
      const std::string msg = std::string("NCCL asynchronous error on group ") + std::to_string(kv.first) +
                              ": " + ncclGetErrorString(async);
      for (auto& c : comms_)
        if (c.second) ncclCommAbort(c.second);
      comms_.clear();
      world_ = nullptr;
      throw NcclError(msg + " (communicators aborted)");
    }
  }
}

Comm::~Comm() {
  for (auto& kv : comms_)
    if (kv.second && kv.second != world_) ncclCommDestroy(kv.second);
  if (world_) ncclCommDestroy(world_);
}

ncclComm_t Comm::comm_for(const Group& g) const {
  auto it = comms_.find(g.id);
  if (it == comms_.end())
    throw NcclError("Comm: no communicator for group " + std::to_string(g.id));
  return it->second;
}

void Comm::bcast(const Group& g, int root_rank, void* buf, size_t count, ncclDataType_t t,
                 Category cat, uint64_t words, cudaStream_t s) {
  NvtxRange nvtx_range("comm bcast");
  (void)g.index_of(rank_);
  const int root = g.index_of(root_rank);
  if (g.size() == 1) return;
  if (local_)
    local_->bcast(g, root, buf, count * dtype_size(t), s);
  else if (count)
    CG_NCCL(ncclBroadcast(buf, buf, count, t, root, comm_for(g), s));
  CommCounter& c = ctr(cat);
  c.calls += 1;
  c.payload_words += words;
  if (rank_ == root_rank) {
    c.words_sent += words * (g.size() - 1);
    c.messages += g.size() - 1;
  } else {
    c.words_received += words;
  }
}

void Comm::bcast_csr(const Group& g, int root_rank, int64_t* row_ptr, int64_t n_rows,
                     int32_t* col, float* vals, int64_t nnz, Category cat, cudaStream_t s) {
  NvtxRange nvtx_range("comm bcast_csr");
  (void)g.index_of(rank_);
  const int root = g.index_of(root_rank);
  if (g.size() == 1) return;
  if (local_) {
    local_->bcast3(g, root, row_ptr, static_cast<size_t>(n_rows + 1) * 8, col, static_cast<size_t>(nnz) * 4,
                   vals, static_cast<size_t>(nnz) * 4, s);
  } else {
  ncclComm_t comm = comm_for(g);
  CG_NCCL(ncclGroupStart());
  CG_NCCL(ncclBroadcast(row_ptr, row_ptr, static_cast<size_t>(n_rows + 1), ncclInt64, root, comm, s));
  if (nnz) {
    CG_NCCL(ncclBroadcast(col, col, static_cast<size_t>(nnz), ncclInt32, root, comm, s));
    CG_NCCL(ncclBroadcast(vals, vals, static_cast<size_t>(nnz), ncclFloat32, root, comm, s));
  }
  CG_NCCL(ncclGroupEnd());
  }
  CommCounter& c = ctr(cat);
  const uint64_t words = static_cast<uint64_t>(nnz);
  c.calls += 1;
  c.payload_words += words;
  if (rank_ == root_rank) {
    c.words_sent += words * (g.size() - 1);
    c.messages += g.size() - 1;
  } else {
    c.words_received += words;
  }
}

void Comm::all_reduce(const Group& g, void* buf, size_t count, ncclDataType_t t, Category cat,
                      uint64_t words, cudaStream_t s) {
  NvtxRange nvtx_range("comm all_reduce");
  const int member = g.index_of(rank_);
  if (g.size() == 1) return;
  if (local_)
    local_->all_reduce(g, buf, count, local_dtype(t), s);
  else if (count)
    CG_NCCL(ncclAllReduce(buf, buf, count, t, ncclSum, comm_for(g), s));
  const uint64_t gs = g.size(), m = words, r = static_cast<uint64_t>(member);
  auto chunk = [&](uint64_t j) { return m / gs + (j < m % gs ? 1 : 0); };
  CommCounter& c = ctr(cat);
  c.calls += 1;
  c.payload_words += m;
  c.words_sent += 2 * m - chunk((r + 1) % gs) - chunk((r + 2) % gs);
  c.words_received += 2 * m - chunk(r) - chunk((r + 1) % gs);
  c.messages += 2 * (gs - 1);
}

void Comm::reduce_scatter(const Group& g, const void* send, void* recv, size_t slice_count,
                          ncclDataType_t t, Category cat, const std::vector<uint64_t>& slot_words,
                          cudaStream_t s) {
  NvtxRange nvtx_range("comm reduce_scatter");
  const int member = g.index_of(rank_);
  if (g.size() == 1) return;
  if (local_)
    local_->reduce_scatter(g, send, recv, slice_count, local_dtype(t), s);
  else if (slice_count)
    CG_NCCL(ncclReduceScatter(send, recv, slice_count, t, ncclSum, comm_for(g), s));
  uint64_t m = 0;
  for (uint64_t w : slot_words) m += w;
  const uint64_t slice = slot_words.at(static_cast<size_t>(member));
  CommCounter& c = ctr(cat);
  c.calls += 1;
  c.payload_words += m;
  c.words_sent += m - slice;
  c.words_received += m - slice;
  c.messages += g.size() - 1;
}

void Comm::all_gather(const Group& g, const void* send, void* recv, size_t slice_count,
                      ncclDataType_t t, Category cat, const std::vector<uint64_t>& slot_words,
                      cudaStream_t s) {
  NvtxRange nvtx_range("comm all_gather");
  const int member = g.index_of(rank_);
  if (g.size() == 1) return;
  if (local_)
    local_->all_gather(g, send, recv, slice_count * dtype_size(t), s);
  else if (slice_count)
    CG_NCCL(ncclAllGather(send, recv, slice_count, t, comm_for(g), s));
  uint64_t m = 0;
  for (uint64_t w : slot_words) m += w;
  CommCounter& c = ctr(cat);
  c.calls += 1;
  c.payload_words += m;
  c.words_sent += m - slot_words.at((static_cast<size_t>(member) + 1) % g.size());
  c.words_received += m - slot_words.at(static_cast<size_t>(member));
  c.messages += g.size() - 1;
}

void Comm::bcast_all(const Group& g, void* buf, size_t slice_count, ncclDataType_t t,
                     Category cat, const std::vector<uint64_t>& words, cudaStream_t s) {
  const int member = g.index_of(rank_);
  if (g.size() == 1) return;
  const size_t esize = dtype_size(t);
  char* base = static_cast<char*>(buf);
  if (local_)
    local_->all_gather(g, base + static_cast<size_t>(member) * slice_count * esize, buf, slice_count * esize, s);
  else if (slice_count)
    CG_NCCL(ncclAllGather(base + static_cast<size_t>(member) * slice_count * esize, buf, slice_count,
                          t, comm_for(g), s));
  meter_bcast_all(g, cat, words);
}

void Comm::meter_bcast_all(const Group& g, Category cat, const std::vector<uint64_t>& words) {
  const int member = g.index_of(rank_);
  if (g.size() == 1) return;
  CommCounter& c = ctr(cat);
  for (int q = 0; q < g.size(); ++q) {
    const uint64_t w = words.at(static_cast<size_t>(q));
    c.calls += 1;
    c.payload_words += w;
    if (q == member) {
      c.words_sent += w * (g.size() - 1);
      c.messages += g.size() - 1;
    } else {
      c.words_received += w;
    }
  }
}

void Comm::setup_all_gather(const void* send, void* recv, size_t count, ncclDataType_t t,
                            cudaStream_t s) {
  const size_t bytes = count * dtype_size(t);
  if (local_) {
    local_->setup_all_gather(send, recv, bytes, s);
    return;
  }
  if (ranks_ == 1) {
    if (send != recv) CG_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  CG_NCCL(ncclAllGather(send, recv, count, t, world_, s));
}

}  // namespace cagnet
