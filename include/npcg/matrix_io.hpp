// Matrix file ingestion for the B200 facade (reference: npcg/matrix_io.hpp,
// core/src/matrix_io.cpp:29-248) -- SURVEY 8(f) row f4: files a reference user
// feeds to `npcg solve` load into the same npcg::Matrix the device operators
// take (e.g. DenseOperator(io::load_matrix(path, fmt))).
//
// Formats (same on-disk contract as the reference):
//  * matrix-market: "%%MatrixMarket matrix coordinate real|integer
//    general|symmetric", '%' comments, a size line "rows cols entries", then
//    1-based "i j value" lines; symmetric files hold the lower triangle and
//    are mirrored on load; the entry count must match.
//  * csv-dense: one row per line, comma-separated, every row the same length.
//  * raw-f64: two little-endian uint64 dims (rows, cols), then rows*cols
//    little-endian doubles in row-major order; round-trips bitwise.
// Errors: std::runtime_error "load_matrix - <path>:<line>: <what>" for parse
// failures (the line number of the offending line), std::invalid_argument for
// an unknown format name.
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "types.hpp"

namespace npcg::io {

enum class MatrixFormat { matrix_market, csv_dense, raw_f64 };

inline MatrixFormat parse_format(const std::string& name) {
  static const std::pair<const char*, MatrixFormat> names[] = {
      {"matrix-market", MatrixFormat::matrix_market}, {"csv-dense", MatrixFormat::csv_dense},
      {"raw-f64", MatrixFormat::raw_f64}};
  for (const auto& [n, f] : names)
    if (name == n) return f;
  throw std::invalid_argument("parse_format: unknown format '" + name + "'");
}

inline std::string format_name(MatrixFormat f) {
  switch (f) {
    case MatrixFormat::matrix_market: return "matrix-market";
    case MatrixFormat::csv_dense: return "csv-dense";
    case MatrixFormat::raw_f64: return "raw-f64";
  }
  throw std::invalid_argument("format_name: unknown format");
}

namespace detail {

[[noreturn]] inline void fail_at(const std::string& path, long line, const std::string& what) {
  throw std::runtime_error("load_matrix - " + path + ":" + std::to_string(line) + ": " + what);
}

inline std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// Line reader that counts lines (1-based) for the error messages.
struct Lines {
  std::ifstream in;
  long no = 0;
  explicit Lines(const std::string& path) : in(path) {
    if (!in) throw std::runtime_error("load_matrix - cannot open " + path);
  }
  bool next(std::string& s) {
    if (!std::getline(in, s)) return false;
    ++no;
    return true;
  }
};

inline double max_abs(const Matrix& m) {
  double s = 0.0;
  for (Index k = 0; k < m.size(); ++k) s = std::max(s, std::fabs(m.data()[k]));
  return s;
}

inline bool is_symmetric(const Matrix& m) {
  if (m.rows() != m.cols()) return false;
  const double tol = 1e-12 * std::max(1.0, max_abs(m));
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = j + 1; i < m.rows(); ++i)
      if (std::fabs(m(i, j) - m(j, i)) > tol) return false;
  return true;
}

inline Matrix read_mm(const std::string& path) {
  Lines f(path);
  std::string s;
  if (!f.next(s)) fail_at(path, 1, "empty file");
  std::istringstream head(s);
  std::string tag, object, layout, field, symmetry;
  head >> tag >> object >> layout >> field >> symmetry;
  if (tag != "%%MatrixMarket" || lower(object) != "matrix") fail_at(path, f.no, "expected a MatrixMarket banner");
  if (lower(layout) != "coordinate") fail_at(path, f.no, "only coordinate format is supported");
  if (lower(field) != "real" && lower(field) != "integer")
    fail_at(path, f.no, "only real-valued matrices are supported");
  const std::string sym = lower(symmetry);
  if (sym != "symmetric" && sym != "general") fail_at(path, f.no, "only general or symmetric matrices are supported");
  const bool mirror = sym == "symmetric";
  Index rows = 0, cols = 0;
  long count = -1;
  while (f.next(s)) {
    if (s.empty() || s[0] == '%') continue;
    std::istringstream sz(s);
    if (!(sz >> rows >> cols >> count)) fail_at(path, f.no, "malformed size line");
    break;
  }
  if (count < 0) fail_at(path, f.no, "missing size line");
  if (rows < 1 || cols < 1) fail_at(path, f.no, "dimensions must be positive");
  if (mirror && rows != cols) fail_at(path, f.no, "a symmetric matrix must be square");
  Matrix m(rows, cols);
  long got = 0;
  while (f.next(s)) {
    if (s.empty() || s[0] == '%') continue;
    std::istringstream e(s);
    Index i = 0, j = 0;
    double v = 0.0;
    if (!(e >> i >> j >> v)) fail_at(path, f.no, "malformed entry");
    if (i < 1 || i > rows || j < 1 || j > cols) fail_at(path, f.no, "entry index out of range");
    if (mirror && j > i) fail_at(path, f.no, "symmetric entries must lie on or below the diagonal");
    m(i - 1, j - 1) = v;
    if (mirror) m(j - 1, i - 1) = v;
    ++got;
  }
  if (got != count)
    fail_at(path, f.no, "expected " + std::to_string(count) + " entries, found " + std::to_string(got));
  return m;
}

inline Matrix read_csv(const std::string& path) {
  Lines f(path);
  std::vector<double> vals;
  Index ncols = -1, nrows = 0;
  std::string s;
  while (f.next(s)) {
    if (s.empty()) continue;
    Index c = 0;
    std::size_t pos = 0;
    while (true) {
      const std::size_t comma = s.find(',', pos);
      const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
      const char* b = tok.c_str();
      char* end = nullptr;
      const double v = std::strtod(b, &end);
      while (end && *end && std::isspace(static_cast<unsigned char>(*end))) ++end;
      if (end == b || (end && *end) || tok.empty()) fail_at(path, f.no, "malformed number '" + tok + "'");
      vals.push_back(v);
      ++c;
      if (comma == std::string::npos || comma + 1 == s.size()) break;  // a trailing comma ends the row
      pos = comma + 1;
    }
    if (ncols >= 0 && c != ncols) fail_at(path, f.no, "inconsistent column count");
    ncols = c;
    ++nrows;
  }
  if (nrows == 0) fail_at(path, 1, "empty file");
  Matrix m(nrows, ncols);
  for (Index i = 0; i < nrows; ++i)
    for (Index j = 0; j < ncols; ++j) m(i, j) = vals[static_cast<size_t>(i * ncols + j)];
  return m;
}

inline Matrix read_raw(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("load_matrix - cannot open " + path);
  std::uint64_t dims[2] = {0, 0};
  if (!in.read(reinterpret_cast<char*>(dims), sizeof(dims)))
    throw std::runtime_error("load_matrix - " + path + ": truncated raw-f64 header");
  if (dims[0] < 1 || dims[1] < 1 || dims[0] > (1u << 24) || dims[1] > (1u << 24))
    throw std::runtime_error("load_matrix - " + path + ": implausible raw-f64 dimensions");
  const Index r = static_cast<Index>(dims[0]), c = static_cast<Index>(dims[1]);
  std::vector<double> rm(static_cast<size_t>(r * c));  // row-major payload, one read
  if (!in.read(reinterpret_cast<char*>(rm.data()), static_cast<std::streamsize>(sizeof(double) * rm.size())))
    throw std::runtime_error("load_matrix - " + path + ": truncated raw-f64 payload");
  Matrix m(r, c);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) m(i, j) = rm[static_cast<size_t>(i * c + j)];
  return m;
}

}  // namespace detail

inline Matrix load_matrix(const std::string& path, MatrixFormat format) {
  switch (format) {
    case MatrixFormat::matrix_market: return detail::read_mm(path);
    case MatrixFormat::csv_dense: return detail::read_csv(path);
    case MatrixFormat::raw_f64: return detail::read_raw(path);
  }
  throw std::invalid_argument("load_matrix: unknown format");
}

inline void save_matrix(const std::string& path, const Matrix& m, MatrixFormat format) {
  if (format == MatrixFormat::raw_f64) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("save_matrix - cannot open " + path);
    const std::uint64_t dims[2] = {static_cast<std::uint64_t>(m.rows()), static_cast<std::uint64_t>(m.cols())};
    out.write(reinterpret_cast<const char*>(dims), sizeof(dims));
    std::vector<double> rm(static_cast<size_t>(m.size()));
    for (Index i = 0; i < m.rows(); ++i)
      for (Index j = 0; j < m.cols(); ++j) rm[static_cast<size_t>(i * m.cols() + j)] = m(i, j);
    out.write(reinterpret_cast<const char*>(rm.data()), static_cast<std::streamsize>(sizeof(double) * rm.size()));
    return;
  }
  std::ofstream out(path);
  if (!out) throw std::runtime_error("save_matrix - cannot open " + path);
  out.precision(17);  // 17 significant digits: text round-trips exactly
  if (format == MatrixFormat::csv_dense) {
    for (Index i = 0; i < m.rows(); ++i) {
      for (Index j = 0; j < m.cols(); ++j) out << (j ? "," : "") << m(i, j);
      out << "\n";
    }
    return;
  }
  if (format != MatrixFormat::matrix_market) throw std::invalid_argument("save_matrix: unknown format");
  const bool sym = detail::is_symmetric(m);  // symmetric writer stores the lower triangle
  std::ostringstream body;
  body.precision(17);
  long count = 0;
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = sym ? j : 0; i < m.rows(); ++i)
      if (m(i, j) != 0.0) {
        body << i + 1 << " " << j + 1 << " " << m(i, j) << "\n";
        ++count;
      }
  out << "%%MatrixMarket matrix coordinate real " << (sym ? "symmetric" : "general") << "\n"
      << m.rows() << " " << m.cols() << " " << count << "\n"
      << body.str();
}

inline Vector load_vector(const std::string& path, MatrixFormat format) {
  const Matrix m = load_matrix(path, format);
  if (m.cols() != 1) throw std::runtime_error("load_vector - " + path + ": expected a single column");
  Vector v(m.rows());
  for (Index i = 0; i < m.rows(); ++i) v(i) = m(i, 0);
  return v;
}

inline Matrix require_symmetric(Matrix m, const std::string& context) {
  if (m.rows() != m.cols()) throw std::runtime_error(context + ": matrix must be square");
  if (!detail::is_symmetric(m)) throw std::runtime_error(context + ": matrix is not symmetric");
  return m;
}

}  // namespace npcg::io
