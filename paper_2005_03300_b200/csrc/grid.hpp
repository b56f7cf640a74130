// Partition topology: ceiling-rule blocks (dist_common.cpp:24-43) and the
// 1D / 1.5D / 2D / 3D process grids with their row / column / fiber groups
// (grid.hpp:29-81, grid.cpp:71-189).  Rank numbering is row major; group
// member lists are ascending, which fixes gather concatenation order.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cagnet {

struct BlockRange {
  int64_t begin = 0;
  int64_t end = 0;
  int64_t size() const { return end - begin; }
};

inline int64_t ceil_div_checked(int64_t a, int64_t b) {
  if (b == 0) throw std::invalid_argument("ceil_div: zero divisor");
  return (a + b - 1) / b;
}

inline BlockRange block_range(int64_t n, int parts, int idx) {
  if (parts <= 0 || idx < 0 || idx >= parts)
    throw std::invalid_argument("block_range: part " + std::to_string(idx) + " of " +
                                std::to_string(parts));
  const int64_t step = n == 0 ? 0 : ceil_div_checked(n, parts);
  int64_t b = static_cast<int64_t>(idx) * step;
  if (b > n) b = n;
  int64_t e = b + step;
  if (e > n) e = n;
  return BlockRange{b, e};
}

inline std::vector<int64_t> block_sizes(int64_t n, int parts) {
  std::vector<int64_t> s(static_cast<size_t>(parts));
  for (int i = 0; i < parts; ++i) s[static_cast<size_t>(i)] = block_range(n, parts, i).size();
  return s;
}

enum class StrategyKind : int { OneD = 0, OneFiveD = 1, TwoD = 2, ThreeD = 3 };
enum class GridKind : int { Row1D = 0, Grid15D = 1, Grid2D = 2, Grid3D = 3 };

inline const char* strategy_kind_name(StrategyKind k) {
  switch (k) {
    case StrategyKind::OneD: return "1d";
    case StrategyKind::OneFiveD: return "1.5d";
    case StrategyKind::TwoD: return "2d";
    case StrategyKind::ThreeD: return "3d";
  }
  return "?";
}

// dist.hpp:51-56
struct Strategy {
  StrategyKind kind = StrategyKind::OneD;
  int ranks = 1;
  int repl = 1;
  int block = 0;
};

struct Group {
  int id = 0;
  std::vector<int> members;
  size_t size() const { return members.size(); }
  int index_of(int rank) const {
    for (size_t i = 0; i < members.size(); ++i)
      if (members[i] == rank) return static_cast<int>(i);
    throw std::invalid_argument("Group::index_of: rank " + std::to_string(rank) +
                                " is not a member of group " + std::to_string(id));
  }
};

inline int exact_isqrt(int p, const char* who) {
  int r = 0;
  while ((r + 1) * (r + 1) <= p) ++r;
  if (r * r != p)
    throw std::invalid_argument(std::string(who) + ": " + std::to_string(p) + " is not a perfect square");
  return r;
}
inline int exact_icbrt(int p, const char* who) {
  int r = 0;
  while ((r + 1) * (r + 1) * (r + 1) <= p) ++r;
  if (r * r * r != p)
    throw std::invalid_argument(std::string(who) + ": " + std::to_string(p) + " is not a perfect cube");
  return r;
}

class ProcessGrid {
 public:
  static ProcessGrid make(const Strategy& s) {  // make_grid, dist_common.cpp:55-65
    if (s.block < 0) throw std::invalid_argument("strategy: panel block width must be non-negative");
    if (s.ranks <= 0)
      throw std::invalid_argument("ProcessGrid: rank count " + std::to_string(s.ranks) + " must be positive");
    ProcessGrid g;
    g.ranks_ = s.ranks;
    switch (s.kind) {
      case StrategyKind::OneD:
        g.kind_ = GridKind::Row1D;
        g.rows_ = s.ranks;
        g.cols_ = 1;
        break;
      case StrategyKind::OneFiveD:
        if (s.repl <= 0 || s.ranks % s.repl != 0)
          throw std::invalid_argument("ProcessGrid::grid15d: replication factor " +
                                      std::to_string(s.repl) + " must divide P=" + std::to_string(s.ranks));
        g.kind_ = GridKind::Grid15D;
        g.rows_ = s.ranks / s.repl;
        g.cols_ = s.repl;
        break;
      case StrategyKind::TwoD: {
        const int side = exact_isqrt(s.ranks, "ProcessGrid::grid2d");
        g.kind_ = GridKind::Grid2D;
        g.rows_ = g.cols_ = side;
        break;
      }
      case StrategyKind::ThreeD: {
        const int side = exact_icbrt(s.ranks, "ProcessGrid::grid3d");
        g.kind_ = GridKind::Grid3D;
        g.rows_ = g.cols_ = g.layers_ = side;
        break;
      }
      default:
        throw std::invalid_argument("strategy: unknown kind");
    }
    g.build_groups();
    return g;
  }

  GridKind kind() const { return kind_; }
  int ranks() const { return ranks_; }
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  int layers() const { return layers_; }

  int row_of(int rank) const {
    if (kind_ == GridKind::Grid3D) return (rank % (rows_ * cols_)) / cols_;
    return rank / cols_;
  }
  int col_of(int rank) const { return rank % cols_; }
  int layer_of(int rank) const { return kind_ == GridKind::Grid3D ? rank / (rows_ * cols_) : 0; }
  int rank_at(int row, int col, int layer = 0) const {
    if (row < 0 || row >= rows_ || col < 0 || col >= cols_ || layer < 0 || layer >= layers_)
      throw std::invalid_argument("ProcessGrid::rank_at: coordinates outside the grid");
    return layer * rows_ * cols_ + row * cols_ + col;
  }

  const Group& world() const { return groups_[0]; }
  const Group& row_group(int rank) const { return at(row_of_, rank, "row"); }
  const Group& col_group(int rank) const { return at(col_of_g_, rank, "column"); }
  const Group& fiber_group(int rank) const { return at(fiber_of_, rank, "fiber"); }
  const std::vector<Group>& groups() const { return groups_; }
  bool has_col_groups() const { return kind_ != GridKind::Row1D; }
  bool has_fiber_groups() const { return kind_ == GridKind::Grid3D; }

 private:
  const Group& at(const std::vector<int>& tbl, int rank, const char* what) const {
    const int id = tbl.at(static_cast<size_t>(rank));
    if (id < 0) throw std::invalid_argument(std::string("ProcessGrid: no ") + what + " group on this grid kind");
    return groups_[static_cast<size_t>(id)];
  }

  void build_groups() {
    groups_.clear();
    row_of_.assign(static_cast<size_t>(ranks_), -1);
    col_of_g_.assign(static_cast<size_t>(ranks_), -1);
    fiber_of_.assign(static_cast<size_t>(ranks_), -1);
    auto add = [this](std::vector<int> m) {
      Group g;
      g.id = static_cast<int>(groups_.size());
      g.members = std::move(m);
      groups_.push_back(std::move(g));
      return groups_.back().id;
    };
    std::vector<int> world(static_cast<size_t>(ranks_));
    for (int r = 0; r < ranks_; ++r) world[static_cast<size_t>(r)] = r;
    const int wid = add(world);
    if (kind_ == GridKind::Row1D) {
      for (int r = 0; r < ranks_; ++r) row_of_[static_cast<size_t>(r)] = wid;
      return;
    }
    for (int layer = 0; layer < layers_; ++layer) {
      for (int i = 0; i < rows_; ++i) {
        std::vector<int> m;
        for (int j = 0; j < cols_; ++j) m.push_back(rank_at(i, j, layer));
        const int id = add(m);
        for (int r : m) row_of_[static_cast<size_t>(r)] = id;
      }
      for (int j = 0; j < cols_; ++j) {
        std::vector<int> m;
        for (int i = 0; i < rows_; ++i) m.push_back(rank_at(i, j, layer));
        const int id = add(m);
        for (int r : m) col_of_g_[static_cast<size_t>(r)] = id;
      }
    }
    if (kind_ == GridKind::Grid3D) {
      for (int i = 0; i < rows_; ++i)
        for (int j = 0; j < cols_; ++j) {
          std::vector<int> m;
          for (int k = 0; k < layers_; ++k) m.push_back(rank_at(i, j, k));
          const int id = add(m);
          for (int r : m) fiber_of_[static_cast<size_t>(r)] = id;
        }
    }
  }

  GridKind kind_ = GridKind::Row1D;
  int ranks_ = 1, rows_ = 1, cols_ = 1, layers_ = 1;
  std::vector<Group> groups_;
  std::vector<int> row_of_, col_of_g_, fiber_of_;
};

// ---- tile geometry shared by the trainers and the host-only C-ABI --------------
// 3D sub-block k of vertex block a (dist_3d.cpp:21-25); the whole block when
// the grid has one layer (2D).
inline BlockRange summa_subrows(const ProcessGrid& g, int64_t n, int a, int b) {
  const BlockRange outer = block_range(n, g.rows(), a);
  const BlockRange inner = block_range(outer.size(), g.layers(), b);
  return BlockRange{outer.begin + inner.begin, outer.begin + inner.end};
}

// Trainer*::tile_rows (dist_1d.cpp:20-22, dist_15d.cpp:20-22, dist_2d.cpp:21-23,
// dist_3d.cpp:31-33).
inline BlockRange tile_rows_of(const ProcessGrid& g, int64_t n, int rank) {
  switch (g.kind()) {
    case GridKind::Row1D: return block_range(n, g.ranks(), rank);
    case GridKind::Grid15D: return block_range(n, g.rows(), g.row_of(rank));
    default: return summa_subrows(g, n, g.row_of(rank), g.layer_of(rank));
  }
}

// Trainer*::tile_cols: full width for block-row strategies, column block j otherwise.
inline BlockRange tile_cols_of(const ProcessGrid& g, int rank, int64_t width) {
  if (g.kind() == GridKind::Row1D || g.kind() == GridKind::Grid15D) return BlockRange{0, width};
  return block_range(width, g.cols(), g.col_of(rank));
}

// Trainer15D::tile_owner (dist_15d.cpp:28-30); self elsewhere.
inline int tile_owner_of(const ProcessGrid& g, int rank) {
  return g.kind() == GridKind::Grid15D ? g.rank_at(g.row_of(rank), 0) : rank;
}

}  // namespace cagnet
