// Port of the reference's io_test.cpp KATs (proj/tests/io_test.cpp:29-190)
// against the facade's npcg::io (include/npcg/matrix_io.hpp). Host-only.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>

#include "npcg/matrix_io.hpp"

using namespace npcg;
namespace fs = std::filesystem;

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

static fs::path dir() {
  const auto d = fs::temp_directory_path() / "npcg_b200_io_test";
  fs::create_directories(d);
  return d;
}
static std::string put(const std::string& name, const std::string& text) {
  const auto p = dir() / name;
  std::ofstream(p) << text;
  return p.string();
}
static bool same(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index k = 0; k < a.size(); ++k)
    if (a.data()[k] != b.data()[k]) return false;
  return true;
}
template <class F>
static std::string error_of(F f) {
  try {
    f();
  } catch (const std::runtime_error& e) {
    return std::string("runtime_error:") + e.what();
  } catch (const std::invalid_argument& e) {
    return std::string("invalid_argument:") + e.what();
  }
  return "";
}
static Matrix gaussian(std::mt19937_64& g, Index r, Index c) {
  std::normal_distribution<double> nd;
  Matrix m(r, c);
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = nd(g);
  return m;
}

int main() {
  using io::MatrixFormat;
  {  // symmetric entries are mirrored (:29-40)
    const auto p = put("sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2.0\n2 1 1.0\n2 2 2.0\n");
    const Matrix m = io::load_matrix(p, MatrixFormat::matrix_market);
    Matrix e(2, 2);
    e(0, 0) = 2, e(0, 1) = 1, e(1, 0) = 1, e(1, 1) = 2;
    CHECK(same(m, e));
  }
  {  // general entries verbatim (:42-56)
    const auto p = put("gen.mtx", "%%MatrixMarket matrix coordinate real general\n% a comment line\n2 3 2\n1 2 5.0\n2 1 -1.0\n");
    const Matrix m = io::load_matrix(p, MatrixFormat::matrix_market);
    CHECK(m.rows() == 2 && m.cols() == 3 && m(0, 1) == 5.0 && m(1, 0) == -1.0 && m(0, 0) == 0.0 && m(1, 2) == 0.0);
  }
  {  // parse failures carry the line number (:58-100)
    const auto p = put("count.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n");
    const std::string e = error_of([&] { io::load_matrix(p, MatrixFormat::matrix_market); });
    CHECK(e.find("runtime_error:") == 0 && e.find("expected 3 entries, found 2") != std::string::npos &&
          e.find(":4:") != std::string::npos);
    for (const auto& [name, text] : std::vector<std::pair<std::string, std::string>>{
             {"empty.mtx", ""},
             {"range.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n"},
             {"upper.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n"}}) {
      const auto q = put(name, text);
      CHECK(error_of([&] { io::load_matrix(q, MatrixFormat::matrix_market); }).find("runtime_error:") == 0);
    }
    CHECK(error_of([&] { io::load_matrix((dir() / "nope.mtx").string(), MatrixFormat::matrix_market); })
              .find("runtime_error:") == 0);
  }
  {  // csv parsing is strict (:102-128)
    Matrix e(2, 2);
    e(0, 0) = 1.5, e(0, 1) = 2, e(1, 0) = 3, e(1, 1) = 4;
    CHECK(same(io::load_matrix(put("ok.csv", "1.5,2\n3,4\n"), MatrixFormat::csv_dense), e));
    const auto bad = put("bad.csv", "1,2\n3,x\n");
    CHECK(error_of([&] { io::load_matrix(bad, MatrixFormat::csv_dense); }).find(":2:") != std::string::npos);
    const auto ragged = put("ragged.csv", "1,2\n3\n"), empty = put("empty.csv", "");
    CHECK(error_of([&] { io::load_matrix(ragged, MatrixFormat::csv_dense); }).find("runtime_error:") == 0);
    CHECK(error_of([&] { io::load_matrix(empty, MatrixFormat::csv_dense); }).find("runtime_error:") == 0);
  }
  {  // round trips (:130-162)
    std::mt19937_64 g(11);
    const Matrix a = gaussian(g, 10, 10);
    const auto raw = (dir() / "rt.raw").string();
    io::save_matrix(raw, a, MatrixFormat::raw_f64);
    CHECK(same(io::load_matrix(raw, MatrixFormat::raw_f64), a));
    const Matrix b = gaussian(g, 5, 4);
    const auto csv = (dir() / "rt.csv").string();
    io::save_matrix(csv, b, MatrixFormat::csv_dense);
    CHECK(same(io::load_matrix(csv, MatrixFormat::csv_dense), b));
    const Matrix h = gaussian(g, 6, 6);
    Matrix s(6, 6);
    for (Index i = 0; i < 6; ++i)
      for (Index j = 0; j < 6; ++j) s(i, j) = h(i, j) + h(j, i);
    const auto mtx = (dir() / "rt.mtx").string();
    io::save_matrix(mtx, s, MatrixFormat::matrix_market);
    std::ifstream in(mtx);
    std::string banner;
    std::getline(in, banner);
    CHECK(banner.find("symmetric") != std::string::npos);
    CHECK(same(io::load_matrix(mtx, MatrixFormat::matrix_market), s));
    const Matrix r = gaussian(g, 4, 3);
    const auto gen = (dir() / "rt_gen.mtx").string();
    io::save_matrix(gen, r, MatrixFormat::matrix_market);
    CHECK(same(io::load_matrix(gen, MatrixFormat::matrix_market), r));
  }
  {  // load_vector single columns only (:164-175)
    const auto col = put("col.csv", "1\n2\n3\n"), wide = put("wide.csv", "1,2\n3,4\n");
    const Vector v = io::load_vector(col, MatrixFormat::csv_dense);
    CHECK(v.size() == 3 && v(2) == 3.0);
    CHECK(error_of([&] { io::load_vector(wide, MatrixFormat::csv_dense); }).find("runtime_error:") == 0);
  }
  {  // format names round trip (:177-183)
    for (const char* n : {"matrix-market", "csv-dense", "raw-f64"}) CHECK(io::format_name(io::parse_format(n)) == n);
    CHECK(error_of([] { io::parse_format("hdf5"); }).find("invalid_argument:") == 0);
  }
  {  // require_symmetric guards symmetric slots (:185-...)
    Matrix a(2, 2), b(2, 3);
    a(0, 0) = 1, a(0, 1) = 2, a(1, 0) = 2.5, a(1, 1) = 1;
    CHECK(error_of([&] { io::require_symmetric(a, "solve"); }).find("solve: matrix is not symmetric") !=
          std::string::npos);
    CHECK(error_of([&] { io::require_symmetric(b, "solve"); }).find("solve: matrix must be square") !=
          std::string::npos);
    a(1, 0) = 2;
    CHECK(same(io::require_symmetric(a, "solve"), a));
  }
  if (failures) return 1;
  std::printf("io ok\n");
  return 0;
}
