// Block-row strategies: 1D (dist_1d.cpp:20-89) and 1.5D with replication
// factor c (dist_15d.cpp:20-104).  1D is the c = 1 case of the same code:
// rank (i, j) of the (P/c) x c grid owns block row i, walks the propagation
// stages [chunk_begin(j), chunk_end(j)) (dist_impl.hpp:50-53) broadcasting
// embedding panels down its column group, and the per-column partials meet in
// a row all-reduce.  NCCL broadcast panels are double-buffered on the comm stream
// so stage q+1's NCCL broadcast overlaps stage q's SpMM.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "p2p.hpp"
#include "trainer.hpp"

namespace cagnet {
namespace {

class TrainerRows final : public Trainer {
 public:
  using Trainer::Trainer;

  BlockRange tile_rows(int r) const override { return tile_rows_of(grid_, data_.n, r); }
  BlockRange tile_cols(int r, int64_t width) const override { return tile_cols_of(grid_, r, width); }
  int tile_owner(int r) const override { return tile_owner_of(grid_, r); }

  void distribute() override {
    init_tiles();
    const BlockRange rows = tile_rows(rank_);
    a_parts_.clear();
    at_parts_.clear();
    for (int q = 0; q < blocks(); ++q) {
      const BlockRange cols = block_range(data_.n, blocks(), q);
      a_parts_.push_back(extract_block_device(data_.adj, rows.begin, rows.end, cols.begin, cols.end, cs_));
      at_parts_.push_back(extract_block_device(data_.adj_t, rows.begin, rows.end, cols.begin, cols.end, cs_));
    }
    buf_w_ = 0;
    size_buffers();
    // Coalesced stage panels (and the peer-memory slots) up to 64 columns, or
    // up to the narrow-first panel width when that is narrower.
    coalesce_w_ = std::min<int64_t>(kCoalesceMaxF, padded_ld(big_width()));
    // Coalesced stages: this column's stage panels land side by side in one
    // buffer (one fused NCCL group) and a single SpMM runs over the block row
    // restricted to the stage columns [c_lo, c_hi).
    const int j = grid_.col_of(rank_);
    chunk_ok_ = stage_group().size() > 1 && chunk_end(j) > chunk_begin(j) + 1;
    if (chunk_ok_) {
      c_lo_ = block_range(data_.n, blocks(), chunk_begin(j)).begin;
      c_hi_ = block_range(data_.n, blocks(), chunk_end(j) - 1).end;
      a_chunk_ = extract_block_device(data_.adj, rows.begin, rows.end, c_lo_, c_hi_, cs_);
      at_chunk_ = extract_block_device(data_.adj_t, rows.begin, rows.end, c_lo_, c_hi_, cs_);
      // Rows for whole padded slots (the 1D all-gather writes P equal slots).
      gbuf_.alloc(std::max(c_hi_ - c_lo_, ceil_div64(data_.n, blocks()) * blocks()), coalesce_w_);
      if (one_d() && p2p_enabled_) {
        const size_t bytes = static_cast<size_t>(ceil_div64(data_.n, blocks()) * blocks()) *
                             coalesce_w_ * sizeof(float);
        p2p_ok_ = p2p_.init(*comm_, rank_, grid_.ranks(), device_, bytes, cs_);
        overlap_ok_ = p2p_ok_ && overlap_enabled_;
        if (overlap_ok_) {
          // Own vertex block first in every row (columns relative to c_lo_).
          own_ = block_range(data_.n, blocks(), rank_);
          a_rot_ = rotate_rows_device(a_chunk_, own_.begin - c_lo_, own_.end - c_lo_, cs_);
          at_rot_ = rotate_rows_device(at_chunk_, own_.begin - c_lo_, own_.end - c_lo_, cs_);
        }
      }
    }
    prepare_streams();
    settle();
  }

  void forward_layer(int l) override {
    if (l < 1 || l >= num_layers())
      throw std::invalid_argument("run_forward_layer: layer " + std::to_string(l) + " outside [1, " +
                                  std::to_string(num_layers()) + ")");
    size_buffers();
    const int64_t fin = dims_[static_cast<size_t>(l - 1)];
    const int64_t fout = dims_[static_cast<size_t>(l)];
    const Mat& h = h_[static_cast<size_t>(l - 1)].m;
    Mat z = z_[static_cast<size_t>(l - 1)].m;
    const bool last = l + 1 == num_layers();
    if (reassociate_ && fout < fin) {
      // Narrow-first propagation: Z = Aᵀ (H W) — the same product as
      // (Aᵀ H) W, but the broadcast panels and the SpMM are f_out wide.
      Mat u = view(acc_, h.rows, fout);
      gemm_aw(h, l - 1, 0, 0, u, false, kern::EPI_NONE, Mat{});
      if (!last && fusable(at_parts_, u)) {
        // ReLU in the SpMM's row epilogue: Z and H_l in one pass; when the next
        // layer's exchange moves H_l itself, the epilogue also pushes it
        // straight into the peers' panel buffers.
        kern::SpmmEpi e;
        const Mat& hl = h_[static_cast<size_t>(l)].m;
        e.relu_out = hl.p;
        e.relu_ld = hl.ld;
        const bool next_takes_h =
            l + 1 < num_layers() && !(reassociate_ && dims_[static_cast<size_t>(l + 1)] < dims_[static_cast<size_t>(l)]);
        const bool push = next_takes_h && arm_push(e, hl, /*relu=*/true, u);
        stages(at_parts_, u, z, &e);
        if (push) commit_push();
        return;
      }
      stages(at_parts_, u, z);
      if (!one_d()) row_reduce(z);
      finish_layer(l, z);
      return;
    }
    // A widening layer keeps T = Aᵀ H for the narrow-first backward.
    const bool keep = reassociate_ && fout > fin;
    if (saved_t_.size() < static_cast<size_t>(num_layers())) {
      saved_t_.resize(static_cast<size_t>(num_layers()));
      saved_valid_.assign(static_cast<size_t>(num_layers()), false);
    }
    if (keep && saved_t_[static_cast<size_t>(l)].m.p == nullptr)
      saved_t_[static_cast<size_t>(l)].alloc(h.rows, fin);
    Mat t = keep ? saved_t_[static_cast<size_t>(l)].m : view(acc_, h.rows, fin);
    saved_valid_[static_cast<size_t>(l)] = keep;
    if (fuse_ >= 2 && fout <= kern::kSpmmEpiMaxFo && fusable(at_parts_, h)) {
      // Z = (Aᵀ H) W_l in the SpMM's row epilogue (+ ReLU into H_l; the
      // widening layer also keeps T for the narrow-first backward).
      const Mat& w = W_[static_cast<size_t>(l - 1)].m;
      kern::SpmmEpi e;
      e.W = w.p;
      e.w_sk = w.ld;
      e.w_sn = 1;
      e.fo = static_cast<int>(fout);
      if (keep) {
        e.raw_out = t.p;
        e.raw_ld = t.ld;
      }
      if (!last) {
        e.relu_out = h_[static_cast<size_t>(l)].m.p;
        e.relu_ld = h_[static_cast<size_t>(l)].m.ld;
      }
      stages(at_parts_, h, z, &e);
      if (last) finish_layer(l, z);
      return;
    }
    stages(at_parts_, h, t);
    if (!one_d()) row_reduce(t);
    if (l + 1 == num_layers()) {
      gemm_aw(t, l - 1, 0, 0, z, false, kern::EPI_NONE, Mat{});
      // log_softmax (dense.cpp:94-107) fused with nll_tile (dense.cpp:109-136).
      Mat hl = h_[static_cast<size_t>(l)].m;
      Mat g = g_[static_cast<size_t>(l - 1)].m;
      kern::logsoftmax_nll(z.p, z.rows, static_cast<int>(z.cols), z.ld, 0, static_cast<int>(z.cols), hl.p,
                           hl.ld, g.p, g.ld, labels_.get(), mask_.get(), train_total_,
                           loss_partial_.get(), cs_);
    } else {
      gemm_aw(t, l - 1, 0, 0, z, false, kern::EPI_RELU, h_[static_cast<size_t>(l)].m);
    }
  }

  void backward_and_step() override {
    const int L = num_layers();
    size_buffers();
    // Only column 0 contributes the loss so replicated rows count once.
    if (grid_.col_of(rank_) != 0) kern::zero_bytes(loss_partial_.get(), sizeof(double), cs_);
    loss_all_reduce(loss_partial_.get());
    for (int l = L - 1; l >= 1; --l) {
      const Mat& g = g_[static_cast<size_t>(l - 1)].m;
      if (reassociate_ && saved_t_ok(l)) {
        // Narrow-first backward for a widening layer (f_out > f_in):
        //   Y = Hᵀ (A G) = (Aᵀ H)ᵀ G = Tᵀ G with T kept from the forward pass;
        //   G_prev = (A (G Wᵀ)) ⊙ relu′(Z_prev): the SpMM runs f_in wide.
        Mat y = Y_[static_cast<size_t>(l - 1)].m;
        if (grid_.col_of(rank_) == 0)
          gemm_hts(saved_t_[static_cast<size_t>(l)].m, g, y, false);
        else
          kern::zero_bytes(y.p, y.rows * y.ld * sizeof(float), cs_);
        // Y is only read by the SGD step: its all-reduce runs on the comm
        // stream behind the remaining backward compute (joined before SGD).
        ms_after_cs();
        comm_->all_reduce(grid_.world(), y.p, static_cast<size_t>(y.rows * y.cols), ncclFloat32,
                          Category::Reduce, words(y), ms_);
        if (l >= 2) {
          Mat gp = g_[static_cast<size_t>(l - 2)].m;
          Mat u = view(acc_, g.rows, dims_[static_cast<size_t>(l - 1)]);
          gemm_swt(g, l - 1, 0, 0, u, false, kern::EPI_NONE, nullptr);
          const Mat& zp = z_[static_cast<size_t>(l - 2)].m;
          if (fusable(a_parts_, u)) {
            kern::SpmmEpi e;  // ⊙ relu′(Z_prev) in the SpMM's row epilogue
            e.mask = zp.p;
            e.mask_ld = zp.ld;
            // The next (lower) layer's exchange moves G_prev itself unless it
            // is a narrow-first widening layer (G Wᵀ first): push it directly.
            const bool next_takes_g = l - 1 >= 1 && !(reassociate_ && saved_t_ok(l - 1));
            const bool push = next_takes_g && arm_push(e, gp, /*relu=*/false, u);
            stages(a_parts_, u, gp, &e);
            if (push) commit_push();
            continue;
          }
          stages(a_parts_, u, gp);
          if (!one_d()) row_reduce(gp);
          kern::mask_relu_prime(gp.p, gp.ld, zp.p, zp.ld, gp.rows, gp.cols, cs_);
        }
        continue;
      }
      Mat s = view(acc_, g.rows, dims_[static_cast<size_t>(l)]);
      const int64_t fprev = dims_[static_cast<size_t>(l - 1)];
      bool fused = false;
      if (fuse_ >= 2 && l >= 2 && fprev <= kern::kSpmmEpiMaxFo && fusable(a_parts_, g)) {
        // G_prev = (S Wᵀ) ⊙ relu′(Z_prev) in the SpMM's row epilogue; S itself
        // still lands in `s` for Y = Hᵀ S.
        const Mat& w = W_[static_cast<size_t>(l - 1)].m;
        const Mat& zp = z_[static_cast<size_t>(l - 2)].m;
        Mat gp = g_[static_cast<size_t>(l - 2)].m;
        kern::SpmmEpi e;
        e.W = w.p;
        e.w_sk = 1;
        e.w_sn = w.ld;
        e.fo = static_cast<int>(fprev);
        e.mask = zp.p;
        e.mask_ld = zp.ld;
        e.raw_out = s.p;
        e.raw_ld = s.ld;
        stages(a_parts_, g, gp, &e);
        fused = true;
      } else {
        stages(a_parts_, g, s);
        if (!one_d()) row_reduce(s);
      }
      Mat y = Y_[static_cast<size_t>(l - 1)].m;
      if (grid_.col_of(rank_) == 0)
        gemm_hts(h_[static_cast<size_t>(l - 1)].m, s, y, false);
      else
        kern::zero_bytes(y.p, y.rows * y.ld * sizeof(float), cs_);
      ms_after_cs();
      comm_->all_reduce(grid_.world(), y.p, static_cast<size_t>(y.rows * y.cols), ncclFloat32,
                        Category::Reduce, words(y), ms_);
      if (l >= 2 && !fused) {
        const Mat& zp = z_[static_cast<size_t>(l - 2)].m;
        gemm_swt(s, l - 1, 0, 0, g_[static_cast<size_t>(l - 2)].m, false, kern::EPI_RELU_PRIME, &zp);
      }
    }
    // Peer-memory buffers rotate over consecutive exchanges, and the captured
    // epoch graph repeats its buffer sequence: unless the exchanges per epoch
    // are a multiple of the buffer count, the first exchanges of one epoch
    // would reuse buffers the last ones of the previous epoch still need.
    // Flag-only exchanges pad the count.
    settle_pending();
    while (p2p_ok_ && epoch_exchanges_ % PeerPanels::kBuffers != 0) {
      next_p2p_buffer();
      p2p_.signal(cs_);
      p2p_.wait_ready(cs_);
    }
    cs_after_ms();  // the Y all-reduces
    sgd_all();
  }

  void begin_epoch() override { epoch_exchanges_ = 0; }

  void finish_external_layer() override {
    // A push the layer committed for an exchange that will not come is
    // waited for (device wait count back in step with the publish count),
    // and flag-only exchanges pad the rotation to a multiple of the buffer
    // count, where every epoch starts.
    settle_pending();
    while (p2p_ok_ && p2p_stage_ % PeerPanels::kBuffers != 0) {
      next_p2p_buffer();
      p2p_.signal(cs_);
      p2p_.wait_ready(cs_);
    }
    epoch_exchanges_ = 0;
  }

  void check_async() override {
    // Report both records: the comm world's and the panel exchange's.
    std::string msg;
    try {
      Trainer::check_async();
    } catch (const NcclError& e) {
      msg = e.what();
    }
    try {
      if (p2p_ok_) p2p_.check();
    } catch (const NcclError& e) {
      msg += (msg.empty() ? "" : "; ") + std::string(e.what());
    }
    if (!msg.empty()) throw NcclError(msg);
  }

 private:
  bool one_d() const { return grid_.kind() == GridKind::Row1D; }
  int blocks() const { return grid_.rows(); }
  int repl() const { return grid_.cols(); }
  int chunk_begin(int j) const { return j * (blocks() / repl()); }
  int chunk_end(int j) const { return j + 1 == repl() ? blocks() : (j + 1) * (blocks() / repl()); }
  const Group& stage_group() const { return one_d() ? grid_.world() : grid_.col_group(rank_); }

  static Mat view(OwnedMat& buf, int64_t rows, int64_t cols) {
    return Mat{buf.m.p, rows, cols, padded_ld(cols)};
  }

  // out = sum over this column's stages q of parts[q] * (tile of rank (q, j)).
  // True when stages(parts, mine, out) ends in ONE SpMM whose output is final
  // (1D: no row all-reduce follows) and whose row epilogue can take the next
  // dense step: P = 1, or the coalesced narrow-panel path; f <= 32; one pass.
  bool fusable(const std::vector<DeviceCsr>& parts, const Mat& mine) const {
    if (fuse_ < 1 || !one_d() || mine.cols > kern::kSpmmEpiMaxF) return false;
    if (stage_group().size() == 1 && chunk_end(0) - chunk_begin(0) == 1)
      return spmm_single_pass(parts[static_cast<size_t>(chunk_begin(0))], mine);
    if (chunk_ok_ && mine.ld <= coalesce_w_) {
      const DeviceCsr& blk = &parts == &a_parts_ ? a_chunk_ : at_chunk_;
      return spmm_single_pass(blk, Mat{nullptr, c_hi_ - c_lo_, mine.cols, mine.ld});
    }
    return false;
  }

  void stages(const std::vector<DeviceCsr>& parts, const Mat& mine, Mat out,
              const kern::SpmmEpi* epi = nullptr) {
    if (!(pending_.valid && pending_.src == mine.p)) settle_pending();
    const int j = grid_.col_of(rank_);
    const Group& grp = stage_group();
    const bool comm = grp.size() > 1;
    if (chunk_ok_ && mine.ld <= coalesce_w_) {
      // Narrow panels: latency, not bandwidth, bounds each stage, so the
      // stage broadcasts go out as one NCCL group (same calls, same ledger)
      // into adjacent slots and one SpMM consumes them all.
      const DeviceCsr& blk = &parts == &a_parts_ ? a_chunk_ : at_chunk_;
      Mat g{gbuf_.m.p, c_hi_ - c_lo_, mine.cols, mine.ld};
      if (one_d() && p2p_ok_ && pipelined(parts, mine) && !(epi && epi->W)) {
        // Bandwidth-heavy exchange (Amazon / Protein scale): push the panel to
        // the peers one destination after another (every rank starts with
        // rank + 1), SpMM the own vertex block from the local panel meanwhile,
        // then each peer's column block as its slot lands (rank - 1 first),
        // accumulating; the fused row epilogue rides on the last block.
        const int P = blocks();
        const int64_t step = ceil_div64(data_.n, P);
        const int b = next_p2p_buffer();
        float* base = p2p_.buffer(b);
        std::vector<uint64_t> words;
        for (int q = 0; q < P; ++q)
          words.push_back(static_cast<uint64_t>(block_range(data_.n, P, q).size() * mine.cols));
        comm_->meter_bcast_all(grp, Category::DBcast, words);
        ms_after_cs();
        for (int d = 1; d < P; ++d)
          p2p_.publish_to(b, (rank_ + d) % P, mine.p, mine.ld, mine.rows, mine.cols, step * mine.ld, mine.ld,
                          d + 1 == P, ms_);
        spmm(parts[static_cast<size_t>(rank_)], mine, out, false, nullptr);
        for (int d = 1; d < P; ++d) {
          const int q = (rank_ - d + P) % P;
          const DeviceCsr& part = parts[static_cast<size_t>(q)];
          p2p_.wait_slot(q, cs_);
          const Mat slot{base + q * step * mine.ld, part.n_cols, mine.cols, mine.ld};
          spmm(part, slot, out, true, d + 1 == P ? epi : nullptr);
        }
        p2p_.wait_ready(cs_);
        cs_after_ms();  // pushes done before anything overwrites `mine`
        return;
      }
      if (one_d() && p2p_ok_ && overlap_ok_ && spmm_single_pass(blk, Mat{nullptr, c_hi_ - c_lo_, mine.cols, mine.ld}) &&
          !(epi && epi->W)) {
        // Peer-memory stage with overlap: the pushes to the peers run on the
        // comm stream while this stream SpMMs the own vertex block straight
        // from the local panel (rows rotated so those columns come first),
        // then the remaining columns from the filled buffer, accumulating,
        // with the fused row epilogue on that last pass.
        const int64_t step = ceil_div64(data_.n, blocks());
        const int b = next_p2p_buffer();
        Mat pg{p2p_.buffer(b), c_hi_ - c_lo_, mine.cols, mine.ld};
        std::vector<uint64_t> words;
        for (int q = 0; q < blocks(); ++q)
          words.push_back(static_cast<uint64_t>(block_range(data_.n, blocks(), q).size() * mine.cols));
        comm_->meter_bcast_all(grp, Category::DBcast, words);
        const RotatedCsr& rot = &parts == &a_parts_ ? a_rot_ : at_rot_;
        const double own_share = static_cast<double>(own_.size()) / static_cast<double>(std::max<int64_t>(blk.n_cols, 1));
        const int64_t own_nnz = static_cast<int64_t>(own_share * static_cast<double>(blk.nnz));
        ms_after_cs();
        p2p_.publish(b, mine.p, mine.ld, mine.rows, mine.cols, step * mine.ld, mine.ld, /*skip_self=*/true, ms_);
        // Column c of the block row is row c - own.begin of the local panel.
        const Mat own_panel{mine.p - (own_.begin - c_lo_) * mine.ld, mine.rows, mine.cols, mine.ld};
        spmm_seg(blk.n_rows, own_nnz, blk.row_ptr.get(), rot.mid.get(), rot.col_idx.get(), rot.vals.get(),
                 own_panel, out, false, nullptr, "spmm_own");
        p2p_.wait_ready(cs_);
        cs_after_ms();  // own pushes done before anything overwrites `mine`
        spmm_seg(blk.n_rows, blk.nnz - own_nnz, rot.mid.get(), blk.row_ptr.get() + 1, rot.col_idx.get(),
                 rot.vals.get(), pg, out, true, epi, "spmm");
        return;
      }
      ms_after_cs();
      const int own = one_d() ? rank_ : grid_.row_of(rank_);
      if (own >= chunk_begin(j) && own < chunk_end(j) && !(one_d() && p2p_ok_)) {
        const BlockRange r = block_range(data_.n, blocks(), own);
        kern::copy2d(g.p + (r.begin - c_lo_) * g.ld, g.ld, mine.p, mine.ld, mine.rows, mine.cols, ms_);
      }
      if (one_d() && p2p_ok_) {
        // NVLink peer-memory exchange: push this rank's panel into every
        // rank's buffer (unless the producer kernel already did), wait for
        // the peers' panels, SpMM.
        const int64_t step = ceil_div64(data_.n, blocks());
        const bool pushed = pending_.valid && pending_.src == mine.p && pending_.ld == mine.ld;
        int b;
        if (pushed) {
          b = pending_.buf;
          pending_.valid = false;
        } else {
          settle_pending();
          b = next_p2p_buffer();
        }
        Mat pg{p2p_.buffer(b), c_hi_ - c_lo_, mine.cols, mine.ld};
        std::vector<uint64_t> words;
        for (int q = 0; q < blocks(); ++q)
          words.push_back(static_cast<uint64_t>(block_range(data_.n, blocks(), q).size() * mine.cols));
        comm_->meter_bcast_all(grp, Category::DBcast, words);
        if (!pushed)
          p2p_.publish(b, mine.p, mine.ld, mine.rows, mine.cols, step * mine.ld, mine.ld, /*skip_self=*/false, cs_);
        p2p_.wait_ready(cs_);
        spmm(blk, pg, out, false, epi);
        return;
      }
      if (one_d()) {
        // 1D: every rank roots one stage, so the P broadcasts are an
        // all-gather of the panel slots (ceil-rule blocks = equal padded slots).
        const int64_t step = ceil_div64(data_.n, blocks());
        std::vector<uint64_t> words;
        for (int q = 0; q < blocks(); ++q)
          words.push_back(static_cast<uint64_t>(block_range(data_.n, blocks(), q).size() * g.cols));
        comm_->bcast_all(grp, g.p, static_cast<size_t>(step * g.ld), ncclFloat32, Category::DBcast, words, ms_);
      } else {
        comm_->group_start();
        for (int q = chunk_begin(j); q < chunk_end(j); ++q) {
          const BlockRange r = block_range(data_.n, blocks(), q);
          const int root = grid_.rank_at(q, j);
          bcast_mat(grp, root, Mat{g.p + (r.begin - c_lo_) * g.ld, r.size(), g.cols, g.ld}, Category::DBcast);
        }
        comm_->group_end();
      }
      cs_after_ms();
      spmm(blk, g, out, false, epi);
      return;
    }
    if (epi && !(chunk_end(j) - chunk_begin(j) == 1 && !comm))
      throw std::logic_error("stages: fused epilogue on a multi-stage propagation");
    ms_after_cs();
    int idx = 0;
    for (int q = chunk_begin(j); q < chunk_end(j); ++q, ++idx) {
      const int root = one_d() ? q : grid_.rank_at(q, j);
      const int b = idx & 1;
      Mat panel = root == rank_ ? mine
                                : Mat{panel_[b].m.p, parts[static_cast<size_t>(q)].n_cols, mine.cols, mine.ld};
      if (comm) {
        if (idx >= 2) CG_CUDA(cudaStreamWaitEvent(ms_, ev_free_[b], 0));
        bcast_mat(grp, root, panel, Category::DBcast);
        CG_CUDA(cudaEventRecord(ev_ready_[b], ms_));
        CG_CUDA(cudaStreamWaitEvent(cs_, ev_ready_[b], 0));
      }
      spmm(parts[static_cast<size_t>(q)], panel, out, idx > 0, epi);
      if (comm) CG_CUDA(cudaEventRecord(ev_free_[b], cs_));
    }
    if (idx == 0) kern::zero_bytes(out.p, out.rows * out.ld * sizeof(float), cs_);
  }

  // Activation of a finished pre-activation tile: ReLU, or the fused
  // log_softmax + NLL on the output layer.
  void finish_layer(int l, const Mat& z) {
    Mat hl = h_[static_cast<size_t>(l)].m;
    if (l + 1 == num_layers()) {
      Mat g = g_[static_cast<size_t>(l - 1)].m;
      kern::logsoftmax_nll(z.p, z.rows, static_cast<int>(z.cols), z.ld, 0, static_cast<int>(z.cols), hl.p,
                           hl.ld, g.p, g.ld, labels_.get(), mask_.get(), train_total_,
                           loss_partial_.get(), cs_);
    } else {
      kern::relu(z.p, z.rows, static_cast<int>(z.cols), z.ld, hl.p, hl.ld, cs_);
    }
  }

  void row_reduce(Mat m) {
    ms_after_cs();
    comm_->all_reduce(grid_.row_group(rank_), m.p, static_cast<size_t>(m.rows * m.ld), ncclFloat32,
                      Category::Reduce, words(m), ms_);
    cs_after_ms();
  }

  // Pipelined peer-memory stages pay one SpMM pass per column block, so they
  // are used only when a peer's slot is large enough for the transfer to
  // matter (>= 32 MB: Amazon / Protein, not Reddit) and every per-block SpMM
  // is a single pass.
  bool pipelined(const std::vector<DeviceCsr>& parts, const Mat& mine) const {
    if (!pipeline_enabled_ || blocks() < 2) return false;
    const double slot = static_cast<double>(ceil_div64(data_.n, blocks())) * mine.ld * 4.0;
    const char* e = std::getenv("CAGNET_PIPELINE_MIN_MB");  // tests lower it
    if (slot < (e ? std::atof(e) : 32.0) * 1048576.0) return false;
    for (const DeviceCsr& p : parts)
      if (!spmm_single_pass(p, Mat{nullptr, p.n_cols, mine.cols, mine.ld})) return false;
    return true;
  }

  bool saved_t_ok(int l) const {
    return static_cast<size_t>(l) < saved_valid_.size() && saved_valid_[static_cast<size_t>(l)];
  }

  static constexpr int64_t kCoalesceMaxF = 64;
  int64_t coalesce_w_ = kCoalesceMaxF;  // widest coalesced panel (gbuf_ / peer slots), fixed at distribute
  int64_t buf_w_ = 0;                   // width acc_ / panel_ are sized for

  // acc_ / panel_ sized for big_width() (grown, eagerly, when a
  // propagation-order switch widens them).
  void size_buffers() {
    const int64_t w = big_width();
    if (w <= buf_w_) return;
    acc_.alloc(tile_rows(rank_).size(), w);
    for (int i = 0; i < 2; ++i) panel_[i].alloc(ceil_div64(data_.n, blocks()), w);
    buf_w_ = w;
    CG_CUDA(cudaStreamSynchronize(nullptr));  // the zeroing memsets ran on the legacy stream
  }

  OwnedMat acc_;
  OwnedMat panel_[2];
  bool chunk_ok_ = false;
  int64_t c_lo_ = 0, c_hi_ = 0;
  DeviceCsr a_chunk_, at_chunk_;  // block row restricted to this column's stage columns
  OwnedMat gbuf_;                 // stage panels side by side
  PeerPanels p2p_;                // NVLink peer-memory panel exchange (1D)
  bool p2p_ok_ = false;
  bool overlap_ok_ = false;       // own-block SpMM overlaps the peer pushes
  BlockRange own_{0, 0};          // this rank's vertex block (1D)
  RotatedCsr a_rot_, at_rot_;     // chunk CSRs with the own block first per row
  uint64_t p2p_stage_ = 0;        // exchange count (buffer rotation)
  int epoch_exchanges_ = 0;       // peer-memory exchanges in the current epoch
  int next_p2p_buffer() {
    ++epoch_exchanges_;
    return static_cast<int>(p2p_stage_++ % PeerPanels::kBuffers);
  }

  // Direct push (fused producer + exchange): the SpMM whose row epilogue
  // produces the next exchange's panel also stores it into every rank's buffer
  // for that exchange (GEMM producers do not: their short epilogues issue the
  // remote row stores from too few threads — a 16 x 16 GEMM went from 9.5 to
  // 68 us with the push), then p2p_.signal() raises
  // the ready flags and the consuming stages() call skips its publish.  Safe
  // with three rotating buffers: the producer runs no earlier than during
  // exchange s-1 (peers may still read the buffers of s-1 and s-2) and writes
  // the buffer of s, last read at s-3, which every peer finished before it
  // published s-1 (stream order).
  struct PendingPush {
    bool valid = false;
    int buf = 0;
    const float* src = nullptr;
    int64_t ld = 0;
  };
  PendingPush pending_;  // committed: the next exchange of `src` skips its publish
  PendingPush armed_;    // armed: a producer kernel is about to push `src`
  uint64_t armed_at_ = 0;
  int armed_skip_ = 0;

  // `skip` = exchanges the producer itself takes before the pushed one (1 for
  // an SpMM producer whose own exchange still publishes, else 0).
  bool arm(const Mat& panel, bool relu, int skip, kern::PushSpec* ps) {
    if (!(one_d() && p2p_ok_ && chunk_ok_ && !overlap_ok_ && !pipeline_enabled_ &&
          panel.ld <= coalesce_w_ && !armed_.valid))
      return false;
    const int b = static_cast<int>((p2p_stage_ + static_cast<uint64_t>(skip)) % PeerPanels::kBuffers);
    ps->bufs = p2p_.device_buffers(b);
    ps->n = grid_.ranks();
    ps->off = static_cast<int64_t>(rank_) * ceil_div64(data_.n, blocks()) * panel.ld;
    ps->ld = panel.ld;
    ps->relu = relu;
    armed_ = PendingPush{true, b, panel.p, panel.ld};
    armed_at_ = p2p_stage_;
    armed_skip_ = skip;
    return true;
  }
  bool arm_push(kern::SpmmEpi& e, const Mat& panel, bool relu, const Mat& producer_in) {
    const int skip = pending_.valid && pending_.src == producer_in.p ? 0 : 1;
    kern::PushSpec ps;
    if (!arm(panel, relu, skip, &ps)) return false;
    e.push_bufs = ps.bufs;
    e.push_n = ps.n;
    e.push_off = ps.off;
    e.push_ld = ps.ld;
    e.push_relu = ps.relu;
    return true;
  }

  // After the producer kernel: the pushed exchange takes its buffer in the
  // rotation and its ready flags go up.
  void commit_push() {
    settle_pending();  // an earlier push nobody consumed keeps the wait count in step
    if (p2p_stage_ != armed_at_ + static_cast<uint64_t>(armed_skip_))
      throw std::logic_error("direct push: unexpected exchanges between producer and push");
    const int b = next_p2p_buffer();
    if (b != armed_.buf) throw std::logic_error("direct push: buffer rotation mismatch");
    p2p_.signal(cs_);
    pending_ = armed_;
    armed_.valid = false;
  }

  // A pushed exchange that no stage consumed still has to be waited for, so
  // the device-side wait count stays in step with the publish count.
  std::vector<const DeviceCsr*> stream_csrs() const override {
    std::vector<const DeviceCsr*> v = Trainer::stream_csrs();
    if (chunk_ok_) {
      v.push_back(&a_chunk_);
      v.push_back(&at_chunk_);
    }
    return v;
  }
  void settle_pending() {
    if (!pending_.valid) return;
    pending_.valid = false;
    p2p_.wait_ready(cs_);
  }
  std::vector<OwnedMat> saved_t_;  // T = Aᵀ H of widening layers (narrow-first backward)
  std::vector<bool> saved_valid_;
};

}  // namespace

std::unique_ptr<Trainer> make_trainer_rows(const DeviceDataset& data, std::vector<int64_t> dims,
                                           const double* weights, double lr, Strategy strat,
                                           int rank, const ncclUniqueId* id) {
  return std::make_unique<TrainerRows>(data, std::move(dims), weights, lr, strat, rank, id);
}

}  // namespace cagnet
