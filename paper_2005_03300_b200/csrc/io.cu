// Graph ingest: the reference's text formats (dataset.hpp:79-97,
// dataset.cpp:146-307) parsed on the host, then make_dataset on the GPU.
//
//   edge list   one "u v" pair per line, '#' starts a comment, optional
//               header "% n <count>" (else n = max index + 1)
//   features    one CSV row of doubles per vertex
//   labels      "vertex,label" per line ('#' lines skipped), every vertex
//               covered
//
// from_edge_list (csr.cpp:79-92) = sort + unique of the (u, v) pairs (both
// directions when undirected, self pairs once), then the usual device
// normalisation / transpose.  Error messages follow the reference's wording.
#include <algorithm>
#include <cstdint>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "trainer.hpp"

namespace cagnet {

namespace {

struct EdgeFile {
  std::vector<std::pair<int64_t, int64_t>> edges;
  int64_t n = 0;
};

EdgeFile load_edge_list(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_edge_list: cannot open " + path);
  EdgeFile f;
  bool have_n = false;
  int64_t max_index = -1;
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    std::istringstream ls(line);
    std::string tok;
    if (!(ls >> tok)) continue;
    if (tok == "%") {
      std::string key;
      long long value = 0;
      if (!(ls >> key >> value) || key != "n" || value < 0)
        throw std::runtime_error("load_edge_list: bad header at line " + std::to_string(lineno) +
                                 " of " + path);
      f.n = value;
      have_n = true;
      continue;
    }
    std::istringstream pair(line);
    long long u = 0, v = 0;
    if (!(pair >> u >> v) || u < 0 || v < 0)
      throw std::runtime_error("load_edge_list: expected 'u v' at line " + std::to_string(lineno) +
                               " of " + path);
    max_index = std::max<int64_t>(max_index, std::max<int64_t>(u, v));
    f.edges.emplace_back(u, v);
  }
  if (!have_n) f.n = max_index + 1;
  for (const auto& e : f.edges)
    if (e.first >= f.n || e.second >= f.n)
      throw std::runtime_error("load_edge_list: vertex " + std::to_string(std::max(e.first, e.second)) +
                               " outside declared n=" + std::to_string(f.n) + " in " + path);
  return f;
}

std::vector<double> load_features_csv(const std::string& path, int64_t* rows, int64_t* cols) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_features_csv: cannot open " + path);
  std::vector<double> data;
  int64_t r = 0, c = -1;
  std::string line, cell;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    std::istringstream ls(line);
    int64_t k = 0;
    while (std::getline(ls, cell, ',')) {
      try {
        size_t used = 0;
        const double x = std::stod(cell, &used);
        data.push_back(x);
      } catch (const std::exception&) {
        throw std::runtime_error("load_features_csv: bad number '" + cell + "' at line " +
                                 std::to_string(lineno) + " of " + path);
      }
      ++k;
    }
    if (c >= 0 && k != c)
      throw std::runtime_error("load_features_csv: ragged row at line " + std::to_string(lineno) +
                               " of " + path);
    c = k;
    ++r;
  }
  if (r == 0) throw std::runtime_error("load_features_csv: empty file " + path);
  *rows = r;
  *cols = c;
  return data;
}

std::vector<int64_t> load_labels(const std::string& path, int64_t n) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_labels: cannot open " + path);
  std::vector<int64_t> labels(static_cast<size_t>(n), -1);
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string vtx, lab;
    if (!std::getline(ls, vtx, ',') || !std::getline(ls, lab))
      throw std::runtime_error("load_labels: expected 'vertex,label' at line " +
                               std::to_string(lineno) + " of " + path);
    unsigned long long v = 0;
    long long y = 0;
    try {
      v = std::stoull(vtx);
      y = std::stoll(lab);
    } catch (const std::exception&) {
      throw std::runtime_error("load_labels: bad pair at line " + std::to_string(lineno) + " of " + path);
    }
    if (v >= static_cast<unsigned long long>(n))
      throw std::runtime_error("load_labels: vertex " + std::to_string(v) + " outside [0, " +
                               std::to_string(n) + ") at line " + std::to_string(lineno) + " of " + path);
    labels[static_cast<size_t>(v)] = y;
  }
  for (int64_t i = 0; i < n; ++i)
    if (labels[static_cast<size_t>(i)] < 0)
      throw std::runtime_error("load_labels: no label for vertex " + std::to_string(i) + " in " + path);
  return labels;
}

}  // namespace

std::unique_ptr<DeviceDataset> dataset_load(const std::string& edges_path,
                                            const std::string& features_path,
                                            const std::string& labels_path, bool undirected) {
  EdgeFile ef = load_edge_list(edges_path);
  // from_edge_list (csr.cpp:79-92): both directions when undirected, then
  // from_pairs sort + unique (csr.cpp:59-75).
  std::vector<std::pair<int64_t, int64_t>> pairs;
  pairs.reserve(ef.edges.size() * (undirected ? 2 : 1));
  for (const auto& e : ef.edges) {
    pairs.push_back(e);
    if (undirected && e.first != e.second) pairs.emplace_back(e.second, e.first);
  }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  const int64_t n = ef.n;
  std::vector<int64_t> rp(static_cast<size_t>(n + 1), 0), ci;
  ci.reserve(pairs.size());
  for (const auto& pr : pairs) {
    ++rp[static_cast<size_t>(pr.first + 1)];
    ci.push_back(pr.second);
  }
  for (int64_t i = 0; i < n; ++i) rp[static_cast<size_t>(i + 1)] += rp[static_cast<size_t>(i)];

  int64_t fr = 0, fc = 0;
  std::vector<double> features = load_features_csv(features_path, &fr, &fc);
  if (fr != n)
    throw std::runtime_error("load_dataset: " + std::to_string(fr) + " feature rows for n=" +
                             std::to_string(n));
  std::vector<int64_t> labels = load_labels(labels_path, n);
  int64_t max_label = 0;
  for (int64_t y : labels) max_label = std::max(max_label, y);
  return dataset_make(n, rp.data(), ci.empty() ? nullptr : ci.data(), features.data(), fc,
                      labels.data(), nullptr, max_label + 1);
}

}  // namespace cagnet
