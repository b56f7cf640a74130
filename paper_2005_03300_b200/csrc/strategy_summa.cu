// SUMMA strategies: 2D on a √P x √P grid (dist_2d.cpp:21-193) and 3D on a
// ∛P cube (dist_3d.cpp:21-182).  2D is the single-layer case of the cube:
// rank (i, j, k) holds the A tile block-row i x sub-block (j, k); a layer's
// SpMM leaves a full block-row partial that the fiber reduce-scatter splits
// back into tiles (a no-op fiber of one rank in 2D).  Phase 2 sweeps the
// T tiles along the row against the replicated weight slab; the final
// log_softmax needs whole rows, gathered across the row group.
//
// Ceiling-rule block sizes make the natural row layout of a partial identical
// to NCCL's padded equal-count slices, so reduce-scatter and all-gather run
// in place on buffers that merely carry a zeroed tail.
#include <algorithm>
#include <cstring>

#include "kernels.cuh"
#include "trainer.hpp"

namespace cagnet {
namespace {

struct SparsePanel {
  DevBuf<int64_t> row_ptr;
  DevBuf<int32_t> col;
  DevBuf<float> vals;
  int64_t rows = 0, cols = 0, nnz = 0;
};

class TrainerSumma final : public Trainer {
 public:
  using Trainer::Trainer;

  BlockRange tile_rows(int r) const override { return tile_rows_of(grid_, data_.n, r); }
  BlockRange tile_cols(int r, int64_t width) const override { return tile_cols_of(grid_, r, width); }

  void distribute() override {
    init_tiles();
    const int i = grid_.row_of(rank_), j = grid_.col_of(rank_), k = grid_.layer_of(rank_);
    const BlockRange arows = block_range(data_.n, side(), i);
    const BlockRange acols = subrows(j, k);
    a_parts_.clear();
    at_parts_.clear();
    a_parts_.push_back(extract_block_device(data_.adj, arows.begin, arows.end, acols.begin, acols.end, cs_));
    at_parts_.push_back(extract_block_device(data_.adj_t, arows.begin, arows.end, acols.begin, acols.end, cs_));

    // Every rank learns every tile's shape (unmetered setup, like distribute()).
    const int P = grid_.ranks();
    DevBuf<int64_t> mine(4), all(static_cast<size_t>(4 * P));
    const int64_t m4[4] = {a_parts_[0].n_rows, a_parts_[0].n_cols, a_parts_[0].nnz, at_parts_[0].nnz};
    CG_CUDA(cudaMemcpy(mine.get(), m4, sizeof(m4), cudaMemcpyHostToDevice));
    CG_CUDA(cudaStreamSynchronize(nullptr));  // pageable H2D: DMA done before cs_ reads it
    comm_->setup_all_gather(mine.get(), all.get(), 4, ncclInt64, cs_);
    shapes_.assign(static_cast<size_t>(4 * P), 0);
    CG_CUDA(cudaStreamSynchronize(cs_));
    CG_CUDA(cudaMemcpy(shapes_.data(), all.get(), shapes_.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));

    int64_t max_rows = 0, max_nnz = 0, maxf = 0;
    for (int r = 0; r < P; ++r) {
      max_rows = std::max(max_rows, shapes_[static_cast<size_t>(4 * r)]);
      max_nnz = std::max({max_nnz, shapes_[static_cast<size_t>(4 * r + 2)], shapes_[static_cast<size_t>(4 * r + 3)]});
    }
    for (int64_t d : dims_) maxf = std::max(maxf, d);
    for (auto& sp : spanel_) {
      sp.row_ptr.resize(static_cast<size_t>(max_rows + 1));
      sp.col.resize(static_cast<size_t>(max_nnz));
      sp.vals.resize(static_cast<size_t>(max_nnz));
    }
    // Resident sparse panels: the A / Aᵀ tiles of this rank's row group never
    // change, so they move once here (unmetered setup, like distribute())
    // instead of once per SpMM stage (the reference's SBcast).  The dense
    // H / G / T / S panels still move every layer.
    resident_[0].clear();
    resident_[1].clear();
    if (resident_sparse_ && side() > 1) {
      CommCounter saved[kNumCategories];
      comm_->snapshot(saved);
      ms_after_cs();
      for (int o = 0; o < 2; ++o) {
        const DeviceCsr& local = o == 0 ? a_parts_[0] : at_parts_[0];
        for (int q = 0; q < side(); ++q) {
          const int aroot = grid_.rank_at(i, q, k);
          const int64_t* sh = &shapes_[static_cast<size_t>(4 * aroot)];
          SparsePanel sp;
          const int64_t nnz = o == 0 ? sh[2] : sh[3];
          sp.rows = sh[0];
          sp.cols = sh[1];
          sp.nnz = nnz;
          sp.row_ptr.resize(static_cast<size_t>(sh[0] + 1));
          sp.col.resize(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
          sp.vals.resize(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
          if (aroot == rank_) {
            kern::copy_bytes(sp.row_ptr.get(), local.row_ptr.get(), (sh[0] + 1) * sizeof(int64_t), ms_);
            kern::copy_bytes(sp.col.get(), local.col_idx.get(), nnz * sizeof(int32_t), ms_);
            kern::copy_bytes(sp.vals.get(), local.vals.get(), nnz * sizeof(float), ms_);
          }
          comm_->bcast_csr(grid_.row_group(rank_), aroot, sp.row_ptr.get(), sh[0], sp.col.get(),
                           sp.vals.get(), nnz, Category::SBcast, ms_);
          resident_[o].push_back(std::move(sp));
        }
      }
      CG_CUDA(cudaStreamSynchronize(ms_));
      comm_->restore(saved);
      // Packed streams of the resident tiles: tile q is block (i, (q, k)) of
      // A / Aᵀ, the rows of block row i and the columns subrows(q, k).
      for (int o = 0; o < 2; ++o)
        for (int q = 0; q < side(); ++q) {
          const SparsePanel& sp = resident_[o][static_cast<size_t>(q)];
          build_packed(sp.rows, sp.cols, sp.nnz, sp.row_ptr.get(), sp.col.get(), sp.vals.get(), arows.begin,
                       subrows(q, k).begin);
        }
    }

    int64_t maxall = 0;
    for (int64_t d : dims_) maxall = std::max(maxall, d);
    const int64_t fmax_cols = ceil_div64(maxall, side());
    strip_.alloc(fmax_cols, fmax_cols, fmax_cols);  // Y strips: f_in / √P x f_out / √P
    buf_w_ = 0;
    size_buffers();
    prepare_streams();
    settle();
  }

  // The n-proportional panels sized for big_width() (grown, eagerly, when a
  // propagation-order switch widens them).
  void size_buffers() {
    const int64_t w = big_width();
    if (w <= buf_w_) return;
    const int64_t step_rows = ceil_div64(std::max<int64_t>(data_.n, 1), side());  // vertex block
    const int64_t sub_step = ceil_div64(std::max<int64_t>(step_rows, 1), layers());
    const int64_t fcols = ceil_div64(w, side());
    // Dense panels hold an H/G tile (sub_step rows) or a T/S tile, with room
    // for every column chunk of a chunked 2D panel at its own padded ld.
    const int64_t chunk_slack = 4 * (strat_.block > 0 ? ceil_div64(fcols, strat_.block) : 1);
    for (auto& p : dpanel_) p.alloc(step_rows, fcols + chunk_slack);
    partial_.alloc(step_rows, fcols, -1, layers() * sub_step);
    tslice_.alloc(sub_step, fcols);
    utile_.alloc(sub_step, fcols);
    pfull_.alloc(sub_step, w);
    redbuf_.alloc(static_cast<int64_t>(side()) * sub_step, fcols);
    gather_.alloc(side() * sub_step, fcols, fcols);
    buf_w_ = w;
    CG_CUDA(cudaStreamSynchronize(nullptr));  // the zeroing memsets ran on the legacy stream
  }

  void forward_layer(int l) override {
    if (l < 1 || l >= num_layers())
      throw std::invalid_argument("run_forward_layer: layer " + std::to_string(l) + " outside [1, " +
                                  std::to_string(num_layers()) + ")");
    size_buffers();
    const int i = grid_.row_of(rank_), j = grid_.col_of(rank_), k = grid_.layer_of(rank_);
    const int64_t wprev = dims_[static_cast<size_t>(l - 1)], wcur = dims_[static_cast<size_t>(l)];
    const BlockRange blockrow = block_range(data_.n, side(), i);
    const BlockRange prevc = tile_cols(rank_, wprev);
    const BlockRange mycur = tile_cols(rank_, wcur);
    const Mat& h = h_[static_cast<size_t>(l - 1)].m;

    Mat z = z_[static_cast<size_t>(l - 1)].m;
    const bool last = l + 1 == num_layers();
    if (reassociate_ && wcur < wprev) {
      // Narrow-first propagation Z = Aᵀ (H W): the row-group GEMM runs on H
      // first (U tile: the rank's rows x column block j of f_out), so the
      // SUMMA panels and the SpMM are f_out / √P wide instead of f_in / √P.
      Mat u = row_gemm_reduce(h, l, wprev, wcur);
      Mat part{partial_.m.p, blockrow.size(), mycur.size(), padded_ld(mycur.size())};
      propagate(at_parts_[0], /*transpose=*/true, u, chunks(mycur.size()), part);
      meter_partial(part, at_parts_[0], l);
      Mat t = fiber_reduce_scatter(part, i);
      kern::copy2d(z.p, z.ld, t.p, t.ld, t.rows, t.cols, cs_);
      if (!last)
        kern::relu(z.p, z.rows, static_cast<int>(z.cols), z.ld, h_[static_cast<size_t>(l)].m.p,
                   h_[static_cast<size_t>(l)].m.ld, cs_);
    } else {
      // Phase 1: partial = sum_q At[i, (q,k)] * H[(q,k), j]  (chunked panels in 2D).
      Mat part{partial_.m.p, blockrow.size(), prevc.size(), padded_ld(prevc.size())};
      propagate(at_parts_[0], /*transpose=*/true, h, chunks(prevc.size()), part);
      meter_partial(part, at_parts_[0], l);
      Mat t = fiber_reduce_scatter(part, i);
      // A widening layer keeps its T tile for the narrow-first backward
      // (Y = Tᵀ G instead of Hᵀ (A G), see backward_and_step).
      if (saved_t_.size() < static_cast<size_t>(num_layers())) saved_t_.resize(static_cast<size_t>(num_layers()));
      OwnedMat& keep = saved_t_[static_cast<size_t>(l)];
      keep_t_valid(l, reassociate_ && wcur > wprev);
      if (reassociate_ && wcur > wprev) {
        if (keep.m.p == nullptr) keep.alloc(t.rows, t.cols);
        kern::copy2d(keep.m.p, keep.m.ld, t.p, t.ld, t.rows, t.cols, cs_);
      }
      // Phase 2: Z = sum_q T[i, q] * W[F_q, F_j] (+ ReLU into H_l).
      row_gemm(t, l, wprev, mycur, z, !last, h_[static_cast<size_t>(l)].m);
    }

    if (last) {
      // Whole rows of Z: gather the row group's column tiles (the reference's
      // transpose -> all_gather_rows -> transpose, dist_2d.cpp:120-126).
      const int64_t wmax = ceil_div64(wcur, side());
      const int64_t rows = z.rows;
      float* slot = gather_.m.p + static_cast<int64_t>(j) * rows * wmax;
      kern::copy2d(slot, wmax, z.p, z.ld, rows, z.cols, cs_);
      std::vector<uint64_t> slot_words;
      std::vector<int> widths;
      for (int q = 0; q < side(); ++q) {
        widths.push_back(static_cast<int>(block_range(wcur, side(), q).size()));
        slot_words.push_back(static_cast<uint64_t>(rows * widths.back()));
      }
      ms_after_cs();
      comm_->all_gather(grid_.row_group(rank_), slot, gather_.m.p, static_cast<size_t>(rows * wmax),
                        ncclFloat32, Category::AllGather, slot_words, ms_);
      cs_after_ms();
      Mat hl = h_[static_cast<size_t>(l)].m;
      Mat g = g_[static_cast<size_t>(l - 1)].m;
      kern::logsoftmax_nll_blocks(gather_.m.p, side(), widths.data(), rows * wmax, rows, wmax, j, hl.p,
                                  hl.ld, g.p, g.ld, labels_.get(), mask_.get(), train_total_,
                                  loss_partial_.get(), cs_);
    }
  }

  void backward_and_step() override {
    const int L = num_layers();
    size_buffers();
    const int i = grid_.row_of(rank_), j = grid_.col_of(rank_), k = grid_.layer_of(rank_);
    loss_all_reduce(loss_partial_.get());
    for (int l = L - 1; l >= 1; --l) {
      const int64_t wcur = dims_[static_cast<size_t>(l)], wprev = dims_[static_cast<size_t>(l - 1)];
      const BlockRange blockrow = block_range(data_.n, side(), i);
      const BlockRange mycur = tile_cols(rank_, wcur);
      const BlockRange myprev = tile_cols(rank_, wprev);
      const Mat& g = g_[static_cast<size_t>(l - 1)].m;

      if (reassociate_ && t_valid(l)) {
        narrow_backward(l, g);
        continue;
      }

      // S = A * G with the same split as the forward propagation.
      Mat part{partial_.m.p, blockrow.size(), mycur.size(), padded_ld(mycur.size())};
      propagate(a_parts_[0], /*transpose=*/false, g, {BlockRange{0, mycur.size()}}, part);
      meter_partial(part, a_parts_[0], 0);
      Mat st = fiber_reduce_scatter(part, i);

      // Shared S panel sweep: Y strips (column + fiber all-reduce) and G_prev.
      Mat y = Y_[static_cast<size_t>(l - 1)].m;
      const int64_t step_p = ceil_div64(wprev, side());
      float* yslot = y.p + static_cast<int64_t>(j) * step_p * y.ld;
      Mat gprev = l >= 2 ? g_[static_cast<size_t>(l - 2)].m : Mat{};
      ms_after_cs();
      for (int q = 0; q < side(); ++q) {
        const BlockRange fq = block_range(wcur, side(), q);
        const int sroot = grid_.rank_at(i, q, k);
        const int b = next_buffer();
        Mat spanel = dense_panel(grid_.row_group(rank_), sroot, st, st.rows, fq.size(),
                                 {BlockRange{0, fq.size()}}, b)[0];
        Mat strip{strip_.m.p, myprev.size(), fq.size(), fq.size() > 0 ? fq.size() : 1};
        gemm_hts(h_[static_cast<size_t>(l - 1)].m, spanel, strip, false);
        ms_after_cs();
        comm_->all_reduce(grid_.col_group(rank_), strip.p, static_cast<size_t>(strip.rows * strip.cols),
                          ncclFloat32, Category::Reduce, words(strip), ms_);
        if (grid_.has_fiber_groups())
          comm_->all_reduce(grid_.fiber_group(rank_), strip.p, static_cast<size_t>(strip.rows * strip.cols),
                            ncclFloat32, Category::Reduce, words(strip), ms_);
        cs_after_ms();
        kern::copy2d(yslot + fq.begin, y.ld, strip.p, strip.ld, strip.rows, strip.cols, cs_);
        if (l >= 2) {
          const Mat& zp = z_[static_cast<size_t>(l - 2)].m;
          gemm_swt(spanel, l - 1, myprev.begin, fq.begin, gprev, q > 0,
                   q + 1 == side() ? kern::EPI_RELU_PRIME : kern::EPI_NONE, &zp);
        }
        release_buffer(b);
      }
      std::vector<uint64_t> slot_words;
      for (int q = 0; q < side(); ++q)
        slot_words.push_back(static_cast<uint64_t>(block_range(wprev, side(), q).size() * wcur));
      ms_after_cs();
      comm_->all_gather(grid_.row_group(rank_), yslot, y.p, static_cast<size_t>(step_p * wcur),
                        ncclFloat32, Category::AllGather, slot_words, ms_);
      cs_after_ms();
    }
    sgd_all();
  }

 private:
  void begin_epoch() override { slot_ = 0; }
  // The SUMMA SpMMs stream the resident / broadcast tiles (spmm_raw without a
  // block), never a_parts_ directly: no packed copies.
  std::vector<const DeviceCsr*> stream_csrs() const override { return {}; }
  int64_t buf_w_ = 0;  // width the large panels are sized for
  int side() const { return grid_.rows(); }
  int layers() const { return grid_.layers(); }

  BlockRange subrows(int a, int b) const { return summa_subrows(grid_, data_.n, a, b); }

  std::vector<BlockRange> chunks(int64_t width) const {  // dist_2d.cpp:29-39 (2D only)
    std::vector<BlockRange> out;
    const int64_t b = (grid_.kind() == GridKind::Grid2D && strat_.block > 0) ? strat_.block : 0;
    if (b == 0 || b >= width) {
      out.push_back(BlockRange{0, width});
      return out;
    }
    for (int64_t s = 0; s < width; s += b) out.push_back(BlockRange{s, std::min(s + b, width)});
    return out;
  }

  // dst = sum_q src[rows, F_q] * W_{l-1}[F_q, cols] over the row group: the
  // tiles of src (column blocks F_q of width f_in) are broadcast along the row
  // (DBcast) and multiplied by the replicated weight slab; relu writes
  // relu(dst) to relu_out after the last partial product.
  void row_gemm(const Mat& src, int l, int64_t fin, const BlockRange& cols, Mat dst, bool relu,
                Mat relu_out) {
    const int i = grid_.row_of(rank_), k = grid_.layer_of(rank_);
    int total_calls = 0;
    for (int q = 0; q < side(); ++q) total_calls += static_cast<int>(chunks(block_range(fin, side(), q).size()).size());
    int calls = 0;
    ms_after_cs();
    for (int q = 0; q < side(); ++q) {
      const BlockRange fq = block_range(fin, side(), q);
      const int troot = grid_.rank_at(i, q, k);
      const std::vector<BlockRange> chs = chunks(fq.size());
      const int b = next_buffer();
      std::vector<Mat> pieces = dense_panel(grid_.row_group(rank_), troot, src, src.rows, fq.size(), chs, b);
      for (size_t c = 0; c < chs.size(); ++c) {
        ++calls;
        const int epi = (calls == total_calls && relu) ? kern::EPI_RELU : kern::EPI_NONE;
        gemm_aw(pieces[c], l - 1, fq.begin + chs[c].begin, cols.begin, dst, calls > 1, epi, relu_out);
      }
      release_buffer(b);
    }
    if (total_calls == 0) {
      kern::zero_bytes(dst.p, dst.rows * dst.ld * sizeof(float), cs_);
      if (relu) kern::relu(dst.p, dst.rows, static_cast<int>(dst.cols), dst.ld, relu_out.p, relu_out.ld, cs_);
    }
  }

  // Narrow-first U[rows, F_j(f_out)] = sum_q H[rows, F_q(f_in)] W[F_q, F_j]:
  // every rank multiplies its own H column block by its W row slab for all
  // f_out columns and the row group reduce-scatters the f_out column blocks,
  // so f_out-wide partials move instead of the f_in-wide H tiles.
  Mat row_gemm_reduce(const Mat& h, int l, int64_t fin, int64_t fout) {
    const int j = grid_.col_of(rank_);
    const BlockRange myin = block_range(fin, side(), j);
    const int64_t rows = h.rows;
    const int64_t wslot = ceil_div64(fout, side());
    const int64_t ld = padded_ld(wslot);
    Mat full{pfull_.m.p, rows, fout, padded_ld(fout)};
    gemm_aw(h, l - 1, myin.begin, 0, full, false, kern::EPI_NONE, Mat{});
    if (side() == 1) return full;
    std::vector<uint64_t> slot_words;
    for (int q = 0; q < side(); ++q) {
      const BlockRange oq = block_range(fout, side(), q);
      slot_words.push_back(static_cast<uint64_t>(rows * oq.size()));
      if (oq.size() > 0)
        kern::copy2d(redbuf_.m.p + q * rows * ld, ld, full.p + oq.begin, full.ld, rows, oq.size(), cs_);
    }
    ms_after_cs();
    comm_->reduce_scatter(grid_.row_group(rank_), redbuf_.m.p, utile_.m.p, static_cast<size_t>(rows * ld),
                          ncclFloat32, Category::Reduce, slot_words, ms_);
    cs_after_ms();
    return Mat{utile_.m.p, rows, block_range(fout, side(), j).size(), ld};
  }

  // Narrow-first backward of a widening layer (wcur > wprev), the SUMMA form of
  // the 1D one (strategy_rows.cu):
  //   Y = Hᵀ (A G) = (Aᵀ H)ᵀ G = Tᵀ G with the T tile kept by the forward pass:
  //     the G tiles of the row group are swept like the reference's S panels
  //     (dist_2d.cpp:150-170) and the Y strips meet in the column (+fiber)
  //     all-reduce and the row all-gather;
  //   G_prev = (A (G Wᵀ)) ⊙ relu′(Z_prev): every rank multiplies its G tile by
  //     its W column slab for all f_prev columns, the row group reduce-scatters
  //     the f_prev column blocks, and the SUMMA propagation moves f_prev / √P
  //     wide panels instead of f_cur / √P wide ones.
  void narrow_backward(int l, const Mat& g) {
    const int i = grid_.row_of(rank_), j = grid_.col_of(rank_), k = grid_.layer_of(rank_);
    const int64_t wcur = dims_[static_cast<size_t>(l)], wprev = dims_[static_cast<size_t>(l - 1)];
    const BlockRange blockrow = block_range(data_.n, side(), i);
    const BlockRange mycur = tile_cols(rank_, wcur);
    const BlockRange myprev = tile_cols(rank_, wprev);
    const Mat& t = saved_t_[static_cast<size_t>(l)].m;
    Mat y = Y_[static_cast<size_t>(l - 1)].m;
    const int64_t step_p = ceil_div64(wprev, side());
    float* yslot = y.p + static_cast<int64_t>(j) * step_p * y.ld;
    ms_after_cs();
    for (int q = 0; q < side(); ++q) {
      const BlockRange fq = block_range(wcur, side(), q);
      const int groot = grid_.rank_at(i, q, k);
      const int b = next_buffer();
      Mat gpanel = dense_panel(grid_.row_group(rank_), groot, g, g.rows, fq.size(), {BlockRange{0, fq.size()}}, b)[0];
      Mat strip{strip_.m.p, myprev.size(), fq.size(), fq.size() > 0 ? fq.size() : 1};
      gemm_hts(t, gpanel, strip, false);
      ms_after_cs();
      comm_->all_reduce(grid_.col_group(rank_), strip.p, static_cast<size_t>(strip.rows * strip.cols),
                        ncclFloat32, Category::Reduce, words(strip), ms_);
      if (grid_.has_fiber_groups())
        comm_->all_reduce(grid_.fiber_group(rank_), strip.p, static_cast<size_t>(strip.rows * strip.cols),
                          ncclFloat32, Category::Reduce, words(strip), ms_);
      cs_after_ms();
      kern::copy2d(yslot + fq.begin, y.ld, strip.p, strip.ld, strip.rows, strip.cols, cs_);
      release_buffer(b);
    }
    std::vector<uint64_t> slot_words;
    for (int q = 0; q < side(); ++q)
      slot_words.push_back(static_cast<uint64_t>(block_range(wprev, side(), q).size() * wcur));
    ms_after_cs();
    comm_->all_gather(grid_.row_group(rank_), yslot, y.p, static_cast<size_t>(step_p * wcur),
                      ncclFloat32, Category::AllGather, slot_words, ms_);
    cs_after_ms();
    if (l < 2) return;
    // U tile = sum_q G[rows, F_q(cur)] W[F_j(prev), F_q(cur)]ᵀ over the row group.
    const int64_t rows = g.rows;
    const int64_t wslot = ceil_div64(wprev, side());
    const int64_t ld = padded_ld(wslot);
    Mat full{pfull_.m.p, rows, wprev, padded_ld(wprev)};
    gemm_swt(g, l - 1, 0, mycur.begin, full, false, kern::EPI_NONE, nullptr);
    Mat u = full;
    if (side() > 1) {
      std::vector<uint64_t> red_words;
      for (int q = 0; q < side(); ++q) {
        const BlockRange oq = block_range(wprev, side(), q);
        red_words.push_back(static_cast<uint64_t>(rows * oq.size()));
        if (oq.size() > 0)
          kern::copy2d(redbuf_.m.p + q * rows * ld, ld, full.p + oq.begin, full.ld, rows, oq.size(), cs_);
      }
      ms_after_cs();
      comm_->reduce_scatter(grid_.row_group(rank_), redbuf_.m.p, utile_.m.p, static_cast<size_t>(rows * ld),
                            ncclFloat32, Category::Reduce, red_words, ms_);
      cs_after_ms();
      u = Mat{utile_.m.p, rows, myprev.size(), ld};
    }
    Mat part{partial_.m.p, blockrow.size(), myprev.size(), padded_ld(myprev.size())};
    propagate(a_parts_[0], /*transpose=*/false, u, {BlockRange{0, myprev.size()}}, part);
    meter_partial(part, a_parts_[0], 0);
    Mat st = fiber_reduce_scatter(part, i);
    Mat gprev = g_[static_cast<size_t>(l - 2)].m;
    const Mat& zp = z_[static_cast<size_t>(l - 2)].m;
    kern::copy2d(gprev.p, gprev.ld, st.p, st.ld, st.rows, st.cols, cs_);
    kern::mask_relu_prime(gprev.p, gprev.ld, zp.p, zp.ld, gprev.rows, gprev.cols, cs_);
  }

  // The 3D trainer's SimRuntime gauges (dist_3d.cpp:84-87 forward, 147-150
  // backward): the partial's words, and the resident words = the sparse
  // tile's nonzeros + the partial + the H tiles (those below layer l in the
  // forward pass, fwd_layer > 0; all of them in the backward pass, 0).
  void meter_partial(const Mat& part, const DeviceCsr& tile, int fwd_layer) {
    if (strat_.kind != StrategyKind::ThreeD) return;
    const uint64_t pw = static_cast<uint64_t>(part.rows * part.cols);
    note_prereduction(pw);
    uint64_t resident = static_cast<uint64_t>(tile.nnz) + pw;
    const int upto = fwd_layer > 0 ? fwd_layer : num_layers();
    for (int l2 = 0; l2 < upto; ++l2)
      resident += static_cast<uint64_t>(h_[static_cast<size_t>(l2)].m.rows * h_[static_cast<size_t>(l2)].m.cols);
    note_memory_words(resident);
  }

  void keep_t_valid(int l, bool v) {
    if (t_valid_.size() < static_cast<size_t>(num_layers())) t_valid_.assign(static_cast<size_t>(num_layers()), false);
    t_valid_[static_cast<size_t>(l)] = v;
  }
  bool t_valid(int l) const { return static_cast<size_t>(l) < t_valid_.size() && t_valid_[static_cast<size_t>(l)]; }

  // Double-buffered panel slots: a slot is reused only after the compute
  // stream finished with its previous contents.
  int next_buffer() {
    const int b = static_cast<int>(slot_ & 1);
    if (slot_ >= 2) CG_CUDA(cudaStreamWaitEvent(ms_, ev_free_[b], 0));
    ++slot_;
    return b;
  }
  void release_buffer(int b) { CG_CUDA(cudaEventRecord(ev_free_[b], cs_)); }

  // Broadcasts the column chunks of `src` (root's rows x width tile) over g;
  // returns one contiguous piece per chunk, valid on the compute stream.
  std::vector<Mat> dense_panel(const Group& g, int root, const Mat& src, int64_t rows, int64_t width,
                               const std::vector<BlockRange>& chs, int b) {
    std::vector<Mat> pieces;
    const bool single = chs.size() == 1 && chs[0].begin == 0 && chs[0].end == width;
    float* cursor = dpanel_[b].m.p;
    for (const BlockRange& ch : chs) {
      Mat piece{cursor, rows, ch.size(), padded_ld(ch.size())};
      if (root == rank_) {
        if (single) {
          piece = Mat{src.p, rows, width, src.ld};
        } else {
          kern::copy2d(piece.p, piece.ld, src.p + ch.begin, src.ld, rows, ch.size(), ms_);
        }
      }
      cursor += rows * padded_ld(ch.size());
      if (g.size() > 1) bcast_mat(g, root, piece, Category::DBcast);
      pieces.push_back(piece);
    }
    CG_CUDA(cudaEventRecord(ev_ready_[b], ms_));
    CG_CUDA(cudaStreamWaitEvent(cs_, ev_ready_[b], 0));
    return pieces;
  }

  // out = sum_q A[i, (q,k)] * X[(q,k), j] with A panels broadcast along the
  // row group (SBcast) and X panels down the column group (DBcast).
  void propagate(const DeviceCsr& local, bool transpose, const Mat& mine,
                 const std::vector<BlockRange>& chs, Mat out) {
    const int i = grid_.row_of(rank_), j = grid_.col_of(rank_), k = grid_.layer_of(rank_);
    const Group& row = grid_.row_group(rank_);
    const Group& col = grid_.col_group(rank_);
    ms_after_cs();
    for (int q = 0; q < side(); ++q) {
      const int aroot = grid_.rank_at(i, q, k);
      const int xroot = grid_.rank_at(q, j, k);
      const int b = next_buffer();
      // Sparse panel.
      const int64_t* rp;
      const int32_t* ci;
      const float* vv;
      int64_t arows, acols, annz;
      if (!resident_[transpose ? 1 : 0].empty()) {
        const SparsePanel& sp = resident_[transpose ? 1 : 0][static_cast<size_t>(q)];
        rp = sp.row_ptr.get();
        ci = sp.col.get();
        vv = sp.vals.get();
        arows = sp.rows;
        acols = sp.cols;
        annz = sp.nnz;
      } else if (aroot == rank_) {
        rp = local.row_ptr.get();
        ci = local.col_idx.get();
        vv = local.vals.get();
        arows = local.n_rows;
        acols = local.n_cols;
        annz = local.nnz;
        if (row.size() > 1)
          comm_->bcast_csr(row, aroot, const_cast<int64_t*>(rp), arows, const_cast<int32_t*>(ci),
                           const_cast<float*>(vv), local.nnz, Category::SBcast, ms_);
      } else {
        const int64_t* sh = &shapes_[static_cast<size_t>(4 * aroot)];
        arows = sh[0];
        acols = sh[1];
        const int64_t nnz = transpose ? sh[3] : sh[2];
        annz = nnz;
        comm_->bcast_csr(row, aroot, spanel_[b].row_ptr.get(), arows, spanel_[b].col.get(),
                         spanel_[b].vals.get(), nnz, Category::SBcast, ms_);
        rp = spanel_[b].row_ptr.get();
        ci = spanel_[b].col.get();
        vv = spanel_[b].vals.get();
      }
      // Dense panel: rows of the X tile of rank (q, j, k) = subrows(q, k).
      const int64_t xrows = subrows(q, k).size();
      if (xrows != acols) throw std::logic_error("propagate: panel shapes disagree");
      std::vector<Mat> pieces = dense_panel(col, xroot, mine, xrows, mine.cols, chs, b);
      for (size_t c = 0; c < chs.size(); ++c) {
        Mat dst{out.p + chs[c].begin, out.rows, chs[c].size(), out.ld};
        spmm_raw(arows, annz, rp, ci, vv, pieces[c], dst, q > 0, nullptr, rp != spanel_[b].row_ptr.get());
      }
      release_buffer(b);
    }
  }

  // 3D: reduce-scatter the block-row partial over the fiber (dist_3d.cpp:88);
  // 2D: the partial already is the tile.
  Mat fiber_reduce_scatter(const Mat& part, int i) {
    if (!grid_.has_fiber_groups() || layers() == 1) return part;
    const Group& fiber = grid_.fiber_group(rank_);
    const BlockRange blockrow = block_range(data_.n, side(), i);
    const int64_t sub_step = ceil_div64(std::max<int64_t>(blockrow.size(), 1), layers());
    std::vector<uint64_t> slot_words;
    for (int kk = 0; kk < layers(); ++kk)
      slot_words.push_back(static_cast<uint64_t>(block_range(blockrow.size(), layers(), kk).size() * part.cols));
    ms_after_cs();
    comm_->reduce_scatter(fiber, part.p, tslice_.m.p, static_cast<size_t>(sub_step * part.ld),
                          ncclFloat32, Category::Reduce, slot_words, ms_);
    cs_after_ms();
    return Mat{tslice_.m.p, tile_rows(rank_).size(), part.cols, part.ld};
  }

  std::vector<int64_t> shapes_;
  SparsePanel spanel_[2];
  std::vector<SparsePanel> resident_[2];  // [A, Aᵀ][q]: row-group tiles kept in HBM
  OwnedMat dpanel_[2];
  OwnedMat partial_, tslice_, strip_, gather_, utile_, pfull_, redbuf_;
  std::vector<OwnedMat> saved_t_;  // T = Aᵀ H tiles of widening layers (narrow-first backward)
  std::vector<bool> t_valid_;
  uint64_t slot_ = 0;
};

}  // namespace

std::unique_ptr<Trainer> make_trainer_summa(const DeviceDataset& data, std::vector<int64_t> dims,
                                            const double* weights, double lr, Strategy strat,
                                            int rank, const ncclUniqueId* id) {
  return std::make_unique<TrainerSumma>(data, std::move(dims), weights, lr, strat, rank, id);
}

std::unique_ptr<Trainer> make_trainer_rows(const DeviceDataset& data, std::vector<int64_t> dims,
                                           const double* weights, double lr, Strategy strat,
                                           int rank, const ncclUniqueId* id);

std::unique_ptr<Trainer> make_trainer(const DeviceDataset& data, std::vector<int64_t> dims,
                                      const double* weights, double lr, Strategy strat, int rank,
                                      const ncclUniqueId* id) {
  switch (strat.kind) {
    case StrategyKind::OneD:
    case StrategyKind::OneFiveD:
      return make_trainer_rows(data, std::move(dims), weights, lr, strat, rank, id);
    case StrategyKind::TwoD:
    case StrategyKind::ThreeD:
      return make_trainer_summa(data, std::move(dims), weights, lr, strat, rank, id);
  }
  throw std::invalid_argument("make_trainer: unknown strategy kind");
}

}  // namespace cagnet
