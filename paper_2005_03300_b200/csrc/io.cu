// Graph ingest for load_dataset (dataset.hpp:79-97): the reference's three
// text formats read from a memory-mapped file by all host cores, the edge
// pairs canonicalised on the GPU.
//
//   edge list  "u v" per line; '#' starts a comment; a "% n <count>" header
//              line fixes n (the last one wins), else n = max index + 1
//   features   one comma-separated row of doubles per vertex
//   labels     "vertex,label" per line, '#'-first lines skipped; every
//              vertex needs a non-negative label
//
// Behaviour, not code, follows dataset.cpp:148-307 and csr.cpp:59-92:
// * the file is split into line ranges, one per host thread; each thread
//   scans its lines with the same field semantics as the reference's stream
//   extraction (whitespace-separated unsigned integers with an optional
//   sign; cells converted like std::stod / std::stoull / std::stoll) and
//   records its first failing line, so the error reported is the one the
//   sequential reference would raise first, with the reference's message;
// * from_edge_list's sort + unique of (u, v) pairs (plus mirrored pairs when
//   undirected) runs on the GPU: one 64-bit key u * n + v per pair, a CUB
//   radix sort over the key's significant bits, a unique pass, and the row
//   pointer from a per-row count + scan — then the usual device normalise /
//   transpose of make_dataset.
#include <cub/cub.cuh>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "trainer.hpp"

namespace cagnet {

namespace {

// ---- mapped input ---------------------------------------------------------------------
class MappedFile {
 public:
  MappedFile(const std::string& path, const char* who) {
    fd_ = ::open(path.c_str(), O_RDONLY);
    if (fd_ < 0) throw std::runtime_error(std::string(who) + ": cannot open " + path);
    struct stat st {};
    if (::fstat(fd_, &st) != 0 || S_ISDIR(st.st_mode)) {
      ::close(fd_);
      throw std::runtime_error(std::string(who) + ": cannot open " + path);
    }
    size_ = static_cast<size_t>(st.st_size);
    if (size_) {
      void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
      if (p == MAP_FAILED) {
        ::close(fd_);
        throw std::runtime_error(std::string(who) + ": cannot open " + path);
      }
      data_ = static_cast<const char*>(p);
    }
  }
  ~MappedFile() {
    if (data_) ::munmap(const_cast<char*>(data_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  MappedFile(const MappedFile&) = delete;
  MappedFile& operator=(const MappedFile&) = delete;
  const char* data() const { return data_; }
  size_t size() const { return size_; }

 private:
  int fd_ = -1;
  const char* data_ = nullptr;
  size_t size_ = 0;
};

struct Line {
  const char* b;
  const char* e;  // excludes the '\n'
};

unsigned host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return h ? std::min(h, 64u) : 4u;
}

// Runs fn(t, begin, end) over [0, count) split into contiguous ranges.
template <class F>
void parallel_ranges(size_t count, F&& fn) {
  const unsigned T = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(host_threads(), count / 4096 + 1)));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] { fn(t, count * t / T, count * (t + 1) / T); });
  for (auto& x : th) x.join();
}

// std::getline semantics: lines end at '\n'; a final line without '\n' counts
// when non-empty.  Line boundaries are found by all threads on byte ranges.
std::vector<Line> split_lines(const MappedFile& f) {
  const char* d = f.data();
  const size_t n = f.size();
  std::vector<std::vector<size_t>> nl(host_threads());
  const unsigned T = static_cast<unsigned>(nl.size());
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      const size_t b = n * t / T, e = n * (t + 1) / T;
      for (const char* p = d + b; p < d + e;) {
        const void* q = std::memchr(p, '\n', static_cast<size_t>(d + e - p));
        if (!q) break;
        nl[t].push_back(static_cast<size_t>(static_cast<const char*>(q) - d));
        p = static_cast<const char*>(q) + 1;
      }
    });
  for (auto& x : th) x.join();
  std::vector<Line> lines;
  size_t start = 0;
  for (const auto& v : nl)
    for (size_t pos : v) {
      lines.push_back(Line{d + start, d + pos});
      start = pos + 1;
    }
  if (start < n) lines.push_back(Line{d + start, d + n});
  return lines;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// One unsigned extraction as `istream >> size_t` performs it: skip
// whitespace, optional sign (a minus negates modulo 2^64), decimal digits;
// overflow or no digits fail.
bool scan_unsigned(const char*& p, const char* e, uint64_t* out) {
  while (p < e && is_space(*p)) ++p;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  const char* d0 = p;
  uint64_t v = 0;
  for (; p < e && *p >= '0' && *p <= '9'; ++p) {
    const uint64_t dgt = static_cast<uint64_t>(*p - '0');
    if (v > (UINT64_MAX - dgt) / 10) return false;
    v = v * 10 + dgt;
  }
  if (p == d0) return false;
  *out = neg ? (0 - v) : v;
  return true;
}

// Next whitespace-delimited token of [p, e).
bool next_token(const char*& p, const char* e, const char** tb, const char** te) {
  while (p < e && is_space(*p)) ++p;
  if (p == e) return false;
  *tb = p;
  while (p < e && !is_space(*p)) ++p;
  *te = p;
  return true;
}

// A cell converted like std::stod (leading whitespace, longest numeric
// prefix, inf/nan/hex accepted; nothing converted or out of range fail).
bool cell_double(const char* b, const char* e, double* out) {
  char buf[128];
  std::string big;
  const size_t len = static_cast<size_t>(e - b);
  const char* s;
  if (len < sizeof(buf)) {
    std::memcpy(buf, b, len);
    buf[len] = 0;
    s = buf;
  } else {
    big.assign(b, len);
    s = big.c_str();
  }
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s, &end);
  if (end == s || errno == ERANGE) return false;
  *out = v;
  return true;
}

template <class T, T (*Conv)(const char*, char**, int)>
bool cell_integer(const char* b, const char* e, T* out) {
  std::string s(b, e);
  char* end = nullptr;
  errno = 0;
  const T v = Conv(s.c_str(), &end, 10);
  if (end == s.c_str() || errno == ERANGE) return false;
  *out = v;
  return true;
}

// The first failure a thread saw, by line number (the sequential reference
// raises the lowest one).
struct FirstError {
  size_t line = SIZE_MAX;
  std::string msg;
  void set(size_t l, std::string m) {
    if (l < line) {
      line = l;
      msg = std::move(m);
    }
  }
};

[[noreturn]] void raise_first(std::vector<FirstError>& errs) {
  size_t best = 0;
  for (size_t i = 1; i < errs.size(); ++i)
    if (errs[i].line < errs[best].line) best = i;
  throw std::runtime_error(errs[best].msg);
}

bool any_error(const std::vector<FirstError>& errs) {
  for (const auto& e : errs)
    if (e.line != SIZE_MAX) return true;
  return false;
}

// ---- edge list ------------------------------------------------------------------------
struct EdgeList {
  std::vector<uint64_t> u, v;  // file order
  uint64_t n = 0;
};

EdgeList read_edge_list(const std::string& path) {
  MappedFile f(path, "load_edge_list");
  const std::vector<Line> lines = split_lines(f);
  struct Part {
    std::vector<uint64_t> u, v;
    uint64_t max_index = 0;
    size_t header_line = 0;  // last header in the part (1-based line; 0 = none)
    uint64_t header_n = 0;
  };
  const unsigned T = host_threads();
  std::vector<Part> parts(T);
  std::vector<FirstError> errs(T);
  parallel_ranges(lines.size(), [&](unsigned t, size_t b, size_t e) {
    Part& P = parts[t];
    for (size_t i = b; i < e; ++i) {
      const size_t lineno = i + 1;
      const char* lb = lines[i].b;
      const char* le = lines[i].e;
      if (const void* h = std::memchr(lb, '#', static_cast<size_t>(le - lb))) le = static_cast<const char*>(h);
      const char* p = lb;
      const char *tb, *te;
      if (!next_token(p, le, &tb, &te)) continue;  // blank or comment-only
      if (te - tb == 1 && *tb == '%') {
        const char *kb, *ke;
        uint64_t value = 0;
        const bool ok = next_token(p, le, &kb, &ke) && ke - kb == 1 && *kb == 'n' && scan_unsigned(p, le, &value);
        if (!ok) {
          errs[t].set(lineno, "load_edge_list: bad header at line " + std::to_string(lineno) + " of " + path);
          return;
        }
        P.header_line = lineno;
        P.header_n = value;
        continue;
      }
      const char* q = lb;
      uint64_t u = 0, v = 0;
      if (!scan_unsigned(q, le, &u) || !scan_unsigned(q, le, &v)) {
        errs[t].set(lineno, "load_edge_list: expected 'u v' at line " + std::to_string(lineno) + " of " + path);
        return;
      }
      P.max_index = std::max(P.max_index, std::max(u, v));
      P.u.push_back(u);
      P.v.push_back(v);
    }
  });
  if (any_error(errs)) raise_first(errs);
  EdgeList out;
  bool have_n = false;
  uint64_t max_index = 0;
  size_t total = 0;
  for (const Part& P : parts) {
    if (P.header_line) {
      have_n = true;
      out.n = P.header_n;  // parts are in file order: the last header wins
    }
    max_index = std::max(max_index, P.max_index);
    total += P.u.size();
  }
  out.u.reserve(total);
  out.v.reserve(total);
  for (const Part& P : parts) {
    out.u.insert(out.u.end(), P.u.begin(), P.u.end());
    out.v.insert(out.v.end(), P.v.begin(), P.v.end());
  }
  if (!have_n) out.n = total == 0 ? 0 : max_index + 1;
  for (size_t i = 0; i < total; ++i)  // first offending edge in file order
    if (out.u[i] >= out.n || out.v[i] >= out.n)
      throw std::runtime_error("load_edge_list: vertex " + std::to_string(std::max(out.u[i], out.v[i])) +
                               " outside declared n=" + std::to_string(out.n) + " in " + path);
  return out;
}

// ---- features CSV ------------------------------------------------------------------------
// std::getline(ls, cell, ',') cells of a line: split at commas, an empty
// final cell (trailing comma) is not produced.
template <class F>
bool for_cells(const char* b, const char* e, F&& fn) {
  const char* p = b;
  while (p < e) {
    const char* c = static_cast<const char*>(std::memchr(p, ',', static_cast<size_t>(e - p)));
    const char* ce = c ? c : e;
    if (!fn(p, ce)) return false;
    if (!c) break;
    p = c + 1;
  }
  return true;
}

std::vector<double> read_features(const std::string& path, int64_t* rows, int64_t* cols) {
  MappedFile f(path, "load_features_csv");
  const std::vector<Line> lines = split_lines(f);
  std::vector<size_t> data_lines;  // non-empty lines
  for (size_t i = 0; i < lines.size(); ++i)
    if (lines[i].e != lines[i].b) data_lines.push_back(i);
  if (data_lines.empty()) throw std::runtime_error("load_features_csv: empty file " + path);
  // Width of the first row (the reference compares every row with it).
  size_t width = 0;
  for_cells(lines[data_lines[0]].b, lines[data_lines[0]].e, [&](const char*, const char*) {
    ++width;
    return true;
  });
  std::vector<double> out(data_lines.size() * width);
  std::vector<FirstError> errs(host_threads());
  parallel_ranges(data_lines.size(), [&](unsigned t, size_t b, size_t e) {
    for (size_t r = b; r < e; ++r) {
      const Line& L = lines[data_lines[r]];
      const size_t lineno = data_lines[r] + 1;
      size_t k = 0;
      bool bad = false;
      for_cells(L.b, L.e, [&](const char* cb, const char* ce) {
        double x = 0;
        if (!cell_double(cb, ce, &x)) {
          errs[t].set(lineno, "load_features_csv: bad number '" + std::string(cb, ce) + "' at line " +
                                  std::to_string(lineno) + " of " + path);
          bad = true;
          return false;
        }
        if (k < width) out[r * width + k] = x;
        ++k;
        return true;
      });
      if (bad) return;
      if (k != width) {
        errs[t].set(lineno, "load_features_csv: ragged row at line " + std::to_string(lineno) + " of " + path);
        return;
      }
    }
  });
  if (any_error(errs)) raise_first(errs);
  *rows = static_cast<int64_t>(data_lines.size());
  *cols = static_cast<int64_t>(width);
  return out;
}

// ---- labels --------------------------------------------------------------------------------
std::vector<int64_t> read_labels(const std::string& path, uint64_t n) {
  MappedFile f(path, "load_labels");
  const std::vector<Line> lines = split_lines(f);
  struct Entry {
    uint64_t v;
    int64_t y;
  };
  const unsigned T = host_threads();
  std::vector<std::vector<Entry>> parts(T);
  std::vector<FirstError> errs(T);
  parallel_ranges(lines.size(), [&](unsigned t, size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      const Line& L = lines[i];
      const size_t lineno = i + 1;
      if (L.e == L.b || *L.b == '#') continue;
      const char* comma = static_cast<const char*>(std::memchr(L.b, ',', static_cast<size_t>(L.e - L.b)));
      if (!comma || comma + 1 == L.e) {
        errs[t].set(lineno, "load_labels: expected 'vertex,label' at line " + std::to_string(lineno) + " of " + path);
        return;
      }
      unsigned long long v = 0;
      long long y = 0;
      if (!cell_integer<unsigned long long, std::strtoull>(L.b, comma, &v) ||
          !cell_integer<long long, std::strtoll>(comma + 1, L.e, &y)) {
        errs[t].set(lineno, "load_labels: bad pair at line " + std::to_string(lineno) + " of " + path);
        return;
      }
      if (v >= n) {
        errs[t].set(lineno, "load_labels: vertex " + std::to_string(v) + " outside [0, " + std::to_string(n) +
                                ") at line " + std::to_string(lineno) + " of " + path);
        return;
      }
      parts[t].push_back(Entry{v, y});
    }
  });
  if (any_error(errs)) raise_first(errs);
  std::vector<int64_t> labels(static_cast<size_t>(n), -1);
  for (const auto& P : parts)
    for (const Entry& en : P) labels[static_cast<size_t>(en.v)] = en.y;  // later lines win
  for (uint64_t i = 0; i < n; ++i)
    if (labels[static_cast<size_t>(i)] < 0)
      throw std::runtime_error("load_labels: no label for vertex " + std::to_string(i) + " in " + path);
  return labels;
}

// ---- from_edge_list on the GPU -------------------------------------------------------------
__global__ void pair_keys_kernel(const uint64_t* __restrict__ u, const uint64_t* __restrict__ v, int64_t m,
                                 uint64_t n, bool undirected, uint64_t* __restrict__ keys,
                                 unsigned long long* __restrict__ extra) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = u[i], b = v[i];
    keys[i] = a * n + b;
    if (undirected && a != b) keys[m + static_cast<int64_t>(atomicAdd(extra, 1ull))] = b * n + a;
  }
}

__global__ void row_counts_kernel(const uint64_t* __restrict__ keys, const int* __restrict__ count, uint64_t n,
                                  int64_t* __restrict__ rows_plus1, int32_t* __restrict__ col, float* __restrict__ val) {
  const int64_t m = *count;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    atomicAdd(reinterpret_cast<unsigned long long*>(rows_plus1 + k / n + 1), 1ull);
    col[i] = static_cast<int32_t>(k % n);
    val[i] = 1.0f;
  }
}

unsigned grid_for_count(int64_t m) {
  const int64_t b = (m + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

// csr.cpp:59-92: unit-valued canonical CSR of the (mirrored) pairs.
DeviceCsr csr_from_pairs_device(const std::vector<uint64_t>& hu, const std::vector<uint64_t>& hv, uint64_t n,
                                bool undirected, cudaStream_t s) {
  const int64_t m = static_cast<int64_t>(hu.size());
  const int64_t cap = undirected ? 2 * m : m;
  DeviceCsr out;
  out.device = current_device();
  out.n_rows = out.n_cols = static_cast<int64_t>(n);
  out.row_ptr.resize(static_cast<size_t>(n + 1));
  kern::zero_bytes(out.row_ptr.get(), (n + 1) * sizeof(int64_t), s);
  if (m == 0) {
    out.col_idx.resize(1);
    out.vals.resize(1);
    CG_CUDA(cudaStreamSynchronize(s));
    return out;
  }
  DevBuf<uint64_t> du(static_cast<size_t>(m)), dv(static_cast<size_t>(m));
  DevBuf<uint64_t> keys(static_cast<size_t>(cap)), sorted(static_cast<size_t>(cap)), uniq(static_cast<size_t>(cap));
  DevBuf<unsigned long long> extra(1);
  DevBuf<int> count(1);
  CG_CUDA(cudaMemcpyAsync(du.get(), hu.data(), m * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  CG_CUDA(cudaMemcpyAsync(dv.get(), hv.data(), m * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  kern::zero_bytes(extra.get(), sizeof(unsigned long long), s);
  pair_keys_kernel<<<grid_for_count(m), 256, 0, s>>>(du.get(), dv.get(), m, n, undirected, keys.get(), extra.get());
  CG_LAUNCH_CHECK();
  unsigned long long mirrored = 0;
  CG_CUDA(cudaMemcpyAsync(&mirrored, extra.get(), sizeof(mirrored), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  const int64_t total = m + static_cast<int64_t>(mirrored);
  require(total < INT32_MAX, "load_dataset: more than 2^31 edge pairs");
  // Keys are < n^2: sort only the significant bits.
  int end_bit = 1;
  while (end_bit < 64 && (n * n - 1) >> end_bit) ++end_bit;
  size_t t1 = 0, t2 = 0;
  CG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys.get(), sorted.get(), static_cast<int>(total), 0, end_bit, s));
  CG_CUDA(cub::DeviceSelect::Unique(nullptr, t2, sorted.get(), uniq.get(), count.get(), static_cast<int>(total), s));
  DevBuf<char> tmp(std::max(t1, t2));
  CG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), t1, keys.get(), sorted.get(), static_cast<int>(total), 0, end_bit, s));
  CG_CUDA(cub::DeviceSelect::Unique(tmp.get(), t2, sorted.get(), uniq.get(), count.get(), static_cast<int>(total), s));
  int nnz = 0;
  CG_CUDA(cudaMemcpyAsync(&nnz, count.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  CG_CUDA(cudaStreamSynchronize(s));
  out.nnz = nnz;
  out.col_idx.resize(static_cast<size_t>(std::max(nnz, 1)));
  out.vals.resize(static_cast<size_t>(std::max(nnz, 1)));
  row_counts_kernel<<<grid_for_count(nnz), 256, 0, s>>>(uniq.get(), count.get(), n, out.row_ptr.get(),
                                                        out.col_idx.get(), out.vals.get());
  CG_LAUNCH_CHECK();
  size_t t3 = 0;
  CG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t3, out.row_ptr.get() + 1, out.row_ptr.get() + 1,
                                        static_cast<int64_t>(n), s));
  DevBuf<char> tmp3(t3);
  CG_CUDA(cub::DeviceScan::InclusiveSum(tmp3.get(), t3, out.row_ptr.get() + 1, out.row_ptr.get() + 1,
                                        static_cast<int64_t>(n), s));
  CG_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace

DeviceCsr csr_from_edges_device(int64_t n, int64_t m, const int64_t* u, const int64_t* v, bool undirected,
                                cudaStream_t s) {
  // from_edge_list's validation (csr.cpp:79-92), same message.
  std::vector<uint64_t> hu(static_cast<size_t>(m)), hv(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || v[i] < 0 || u[i] >= n || v[i] >= n)
      throw std::invalid_argument("from_edge_list: edge " + std::to_string(i) + " = (" + std::to_string(u[i]) +
                                  ", " + std::to_string(v[i]) + ") outside vertex range [0, " + std::to_string(n) +
                                  ")");
    hu[static_cast<size_t>(i)] = static_cast<uint64_t>(u[i]);
    hv[static_cast<size_t>(i)] = static_cast<uint64_t>(v[i]);
  }
  require(n >= 0 && n <= INT32_MAX, "from_edge_list: n outside the device's 32-bit column range");
  return csr_from_pairs_device(hu, hv, static_cast<uint64_t>(n), undirected, s);
}

// ---- binary dataset cache ------------------------------------------------------------------
// "CAGNETD1" | int64 {n, f, num_classes, train_count, nnz_adj, nnz_adj_t} |
// adj {row_ptr int64[n+1], col int32[nnz], vals f32[nnz]} | adj_t likewise |
// features f32[n x f] (dense) | labels int32[n] | mask uint8[n].  Host byte
// order; a finished GraphDataset (normalised adjacency and its transpose), so
// loading is a mapped read and the uploads — no generation, no sort.
namespace {
constexpr char kCacheMagic[8] = {'C', 'A', 'G', 'N', 'E', 'T', 'D', '1'};

void write_all(FILE* fp, const void* p, size_t bytes, const std::string& path) {
  if (bytes && std::fwrite(p, 1, bytes, fp) != bytes) throw std::runtime_error("save_dataset: write failed for " + path);
}

template <class T>
std::vector<T> download(const T* dev, size_t count) {
  std::vector<T> h(count);
  if (count) CG_CUDA(cudaMemcpy(h.data(), dev, count * sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}
}  // namespace

void dataset_save(const DeviceDataset& d, const std::string& path) {
  CG_CUDA(cudaSetDevice(d.device));
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw std::runtime_error("save_dataset: cannot open " + path);
  try {
    write_all(fp, kCacheMagic, sizeof(kCacheMagic), path);
    const int64_t hdr[6] = {d.n, d.f, d.num_classes, d.train_count, d.adj.nnz, d.adj_t.nnz};
    write_all(fp, hdr, sizeof(hdr), path);
    for (const DeviceCsr* a : {&d.adj, &d.adj_t}) {
      auto rp = download(a->row_ptr.get(), static_cast<size_t>(a->n_rows + 1));
      auto ci = download(a->col_idx.get(), static_cast<size_t>(a->nnz));
      auto va = download(a->vals.get(), static_cast<size_t>(a->nnz));
      write_all(fp, rp.data(), rp.size() * 8, path);
      write_all(fp, ci.data(), ci.size() * 4, path);
      write_all(fp, va.data(), va.size() * 4, path);
    }
    std::vector<float> feats(static_cast<size_t>(d.n * d.f));
    if (d.n && d.f)
      CG_CUDA(cudaMemcpy2D(feats.data(), d.f * sizeof(float), d.features.get(), d.ldf * sizeof(float),
                           d.f * sizeof(float), d.n, cudaMemcpyDeviceToHost));
    write_all(fp, feats.data(), feats.size() * 4, path);
    auto lab = download(d.labels.get(), static_cast<size_t>(d.n));
    auto msk = download(d.mask.get(), static_cast<size_t>(d.n));
    write_all(fp, lab.data(), lab.size() * 4, path);
    write_all(fp, msk.data(), msk.size(), path);
  } catch (...) {
    std::fclose(fp);
    throw;
  }
  if (std::fclose(fp) != 0) throw std::runtime_error("save_dataset: write failed for " + path);
}

std::unique_ptr<DeviceDataset> dataset_load_binary(const std::string& path, int device) {
  MappedFile f(path, "load_dataset_binary");
  const char* p = f.data();
  size_t left = f.size();
  auto take = [&](size_t bytes) {
    if (bytes > left) throw std::runtime_error("load_dataset_binary: truncated file " + path);
    const char* q = p;
    p += bytes;
    left -= bytes;
    return q;
  };
  if (f.size() < sizeof(kCacheMagic) || std::memcmp(take(sizeof(kCacheMagic)), kCacheMagic, 8) != 0)
    throw std::runtime_error("load_dataset_binary: " + path + " is not a CAGNETD1 dataset cache");
  int64_t hdr[6];
  std::memcpy(hdr, take(sizeof(hdr)), sizeof(hdr));
  const int64_t n = hdr[0], fdim = hdr[1];
  if (n < 0 || n > INT32_MAX || fdim < 0 || hdr[2] <= 0 || hdr[4] < 0 || hdr[5] < 0)
    throw std::runtime_error("load_dataset_binary: corrupt header in " + path);
  // The whole layout is checked against the file size before any device work.
  const uint64_t need = 8 + sizeof(hdr) + 2ull * static_cast<uint64_t>(n + 1) * 8 +
                        static_cast<uint64_t>(hdr[4] + hdr[5]) * 8 + static_cast<uint64_t>(n) * fdim * 4 +
                        static_cast<uint64_t>(n) * 5;
  if (f.size() < need) throw std::runtime_error("load_dataset_binary: truncated file " + path);
  if (f.size() > need) throw std::runtime_error("load_dataset_binary: trailing bytes in " + path);
  CG_CUDA(cudaSetDevice(device));
  auto d = std::make_unique<DeviceDataset>();
  d->device = device;
  d->n = n;
  d->f = fdim;
  d->num_classes = hdr[2];
  d->train_count = hdr[3];
  d->ldf = padded_ld(fdim);
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    for (int w = 0; w < 2; ++w) {
      DeviceCsr& a = w == 0 ? d->adj : d->adj_t;
      const int64_t nnz = hdr[4 + w];
      a.device = device;
      a.n_rows = a.n_cols = n;
      a.nnz = nnz;
      a.row_ptr.resize(static_cast<size_t>(n + 1));
      a.col_idx.resize(static_cast<size_t>(nnz > 0 ? nnz : 1));
      a.vals.resize(static_cast<size_t>(nnz > 0 ? nnz : 1));
      const char* rp = take(static_cast<size_t>(n + 1) * 8);
      const char* ci = take(static_cast<size_t>(nnz) * 4);
      const char* va = take(static_cast<size_t>(nnz) * 4);
      CG_CUDA(cudaMemcpy(a.row_ptr.get(), rp, static_cast<size_t>(n + 1) * 8, cudaMemcpyHostToDevice));
      if (nnz) {
        CG_CUDA(cudaMemcpy(a.col_idx.get(), ci, static_cast<size_t>(nnz) * 4, cudaMemcpyHostToDevice));
        CG_CUDA(cudaMemcpy(a.vals.get(), va, static_cast<size_t>(nnz) * 4, cudaMemcpyHostToDevice));
      }
    }
    d->features.resize(static_cast<size_t>(n * d->ldf > 0 ? n * d->ldf : 1));
    kern::zero_bytes(d->features.get(), static_cast<size_t>(n * d->ldf) * sizeof(float), s);
    CG_CUDA(cudaStreamSynchronize(s));
    const char* fe = take(static_cast<size_t>(n * fdim) * 4);
    if (n && fdim)
      CG_CUDA(cudaMemcpy2D(d->features.get(), d->ldf * sizeof(float), fe, fdim * sizeof(float), fdim * sizeof(float),
                           n, cudaMemcpyHostToDevice));
    d->labels.resize(static_cast<size_t>(n > 0 ? n : 1));
    d->mask.resize(static_cast<size_t>(n > 0 ? n : 1));
    const char* la = take(static_cast<size_t>(n) * 4);
    const char* ma = take(static_cast<size_t>(n));
    if (n) {
      CG_CUDA(cudaMemcpy(d->labels.get(), la, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice));
      CG_CUDA(cudaMemcpy(d->mask.get(), ma, static_cast<size_t>(n), cudaMemcpyHostToDevice));
    }
    // Pageable H2D copies may return before their DMA lands; the dataset's
    // users run on non-blocking streams.
    CG_CUDA(cudaStreamSynchronize(nullptr));
    if (left != 0) throw std::runtime_error("load_dataset_binary: trailing bytes in " + path);
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  CG_CUDA(cudaStreamDestroy(s));
  return d;
}

std::unique_ptr<DeviceDataset> dataset_load(const std::string& edges_path,
                                            const std::string& features_path,
                                            const std::string& labels_path, bool undirected, int device) {
  EdgeList el = read_edge_list(edges_path);
  require(el.n <= static_cast<uint64_t>(INT32_MAX),
          "load_edge_list: n=" + std::to_string(el.n) + " exceeds the device's 32-bit column indices");
  int64_t fr = 0, fc = 0;
  std::vector<double> features = read_features(features_path, &fr, &fc);
  if (static_cast<uint64_t>(fr) != el.n)
    throw std::runtime_error("load_dataset: " + std::to_string(fr) + " feature rows for n=" +
                             std::to_string(el.n));
  std::vector<int64_t> labels = read_labels(labels_path, el.n);
  int64_t max_label = 0;
  for (int64_t y : labels) max_label = std::max(max_label, y);
  CG_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  CG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    DeviceCsr raw = csr_from_pairs_device(el.u, el.v, el.n, undirected, s);
    std::vector<uint64_t>().swap(el.u);
    std::vector<uint64_t>().swap(el.v);
    CG_CUDA(cudaStreamDestroy(s));
    return dataset_make_device(std::move(raw), features.data(), fc, labels.data(), nullptr, max_label + 1);
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
}

}  // namespace cagnet
