// Matrix Market ingest for the sparse / dense operator path (host C++, no GPU).
//
// Restates read_matrix_market / write_matrix_market (proj/include/sssvd/matrix_market.hpp:34-149)
// behind the C ABI so the GPU library reads the same files to the same bits:
//   * header checks in the reference's order (banner, object, field, symmetry; the format is
//     checked after the size line), error text "path:line: what" with the same line counting
//     (comment and blank lines are counted, matrix_market.hpp:57-65);
//   * numbers parsed with std::istringstream >> like the reference (same libstdc++ num_get, so
//     "1.5x" reads 1.5 and "inf"/"nan" are rejected as bad values);
//   * coordinate duplicates summed in file order (Eigen setFromTriplets accumulates each (i, j)
//     left to right in insertion order); explicit zeros are kept as stored entries;
//   * (skew-)symmetric storage expanded; array (skew-)symmetric reads column j from row j down.
// One deliberate deviation: (skew-)symmetric storage of a non-square matrix is rejected with a
// format error, where the reference writes out of bounds.
#include <algorithm>
#include <cctype>
#include <cstdint>
#include <fstream>
#include <iomanip>
#include <memory>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sssvd_gpu.h"

struct sssvd_mm_matrix {
  int64_t rows = 0, cols = 0;
  bool sparse = false;
  std::vector<double> values;  // dense: rows*cols column-major; sparse: nnz
  std::vector<int64_t> colptr, rowind;
};

namespace {

thread_local std::string g_host_error;

struct MmError {
  sssvd_status code;
  std::string what;
};

MmError format_error(const std::string& path, int64_t line, const std::string& what) {
  return {SSSVD_E_FORMAT, path + ":" + std::to_string(line) + ": " + what};
}

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return (char)std::tolower(c); });
  return s;
}

struct Triplet {
  int64_t row, col;
  double value;
};

sssvd_mm_matrix* read_mm(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MmError{SSSVD_E_IO, "read_matrix_market: cannot open " + path};
  int64_t line_no = 1;
  std::string header;
  if (!std::getline(in, header)) throw format_error(path, 1, "empty file");
  std::istringstream hs(header);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket" || lower(object) != "matrix")
    throw format_error(path, 1, "not a MatrixMarket matrix header");
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (field == "complex" || field == "pattern")
    throw format_error(path, 1, "unsupported field '" + field + "' (real data required)");
  if (field != "real" && field != "integer" && field != "double")
    throw format_error(path, 1, "unknown field '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric" && symmetry != "skew-symmetric")
    throw format_error(path, 1, "unsupported symmetry '" + symmetry + "'");
  const bool general = symmetry == "general", skew = symmetry == "skew-symmetric";

  auto next_data_line = [&](std::string& out) {
    while (std::getline(in, out)) {
      ++line_no;
      const auto first = out.find_first_not_of(" \t\r");
      if (first == std::string::npos || out[first] == '%') continue;
      return true;
    }
    return false;
  };

  std::string line;
  if (!next_data_line(line)) throw format_error(path, line_no, "missing size line");
  std::istringstream ls(line);
  auto mm = std::make_unique<sssvd_mm_matrix>();

  if (format == "array") {
    long rows, cols;
    if (!(ls >> rows >> cols) || rows < 1 || cols < 1) throw format_error(path, line_no, "bad array size line");
    if (!general && rows != cols) throw format_error(path, line_no, "symmetric storage needs a square matrix");
    mm->rows = rows;
    mm->cols = cols;
    mm->values.assign((size_t)rows * cols, 0.0);
    for (int64_t j = 0; j < cols; ++j) {
      for (int64_t i = general ? 0 : j; i < rows; ++i) {
        if (!next_data_line(line)) throw format_error(path, line_no, "unexpected end of array data");
        std::istringstream vs(line);
        double value;
        if (!(vs >> value)) throw format_error(path, line_no, "bad array value");
        mm->values[(size_t)j * rows + i] = value;
        if (!general) mm->values[(size_t)i * rows + j] = skew ? -value : value;
      }
    }
    return mm.release();
  }
  if (format != "coordinate") throw format_error(path, 1, "unknown format '" + format + "'");

  long rows, cols, nnz;
  if (!(ls >> rows >> cols >> nnz) || rows < 1 || cols < 1 || nnz < 0)
    throw format_error(path, line_no, "bad coordinate size line");
  if (!general && rows != cols) throw format_error(path, line_no, "symmetric storage needs a square matrix");
  std::vector<Triplet> trip;
  trip.reserve((size_t)nnz * (general ? 1 : 2));
  for (long k = 0; k < nnz; ++k) {
    if (!next_data_line(line)) throw format_error(path, line_no, "unexpected end of coordinate data");
    std::istringstream vs(line);
    long i, j;
    double value;
    if (!(vs >> i >> j >> value)) throw format_error(path, line_no, "bad coordinate entry");
    if (i < 1 || i > rows || j < 1 || j > cols) throw format_error(path, line_no, "index out of range");
    trip.push_back({i - 1, j - 1, value});
    if (!general && i != j) trip.push_back({j - 1, i - 1, skew ? -value : value});
  }
  // compress: stable order by (col, row) keeps file order among duplicates, which are then
  // summed left to right (Eigen setFromTriplets + collapseDuplicates)
  std::vector<size_t> order(trip.size());
  std::iota(order.begin(), order.end(), size_t(0));
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return trip[a].col != trip[b].col ? trip[a].col < trip[b].col : trip[a].row < trip[b].row;
  });
  mm->rows = rows;
  mm->cols = cols;
  mm->sparse = true;
  mm->colptr.assign((size_t)cols + 1, 0);
  for (size_t q = 0; q < order.size(); ++q) {
    const Triplet& t = trip[order[q]];
    if (q > 0 && trip[order[q - 1]].row == t.row && trip[order[q - 1]].col == t.col) {
      mm->values.back() += t.value;
      continue;
    }
    mm->rowind.push_back(t.row);
    mm->values.push_back(t.value);
    ++mm->colptr[(size_t)t.col + 1];
  }
  for (int64_t j = 0; j < cols; ++j) mm->colptr[(size_t)j + 1] += mm->colptr[(size_t)j];
  return mm.release();
}

void write_mm(const std::string& path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* colptr,
              const int64_t* rowind, const double* values, const std::string& comment) {
  std::ofstream out(path);
  if (!out) throw MmError{SSSVD_E_IO, "write_matrix_market: cannot open " + path};
  out << std::setprecision(17);
  if (!colptr) {
    out << "%%MatrixMarket matrix array real general\n";
    if (!comment.empty()) out << "% " << comment << "\n";
    out << rows << " " << cols << "\n";
    for (int64_t e = 0; e < rows * cols; ++e) out << values[e] << "\n";
  } else {
    out << "%%MatrixMarket matrix coordinate real general\n";
    if (!comment.empty()) out << "% " << comment << "\n";
    out << rows << " " << cols << " " << nnz << "\n";
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t k = colptr[j]; k < colptr[j + 1]; ++k) out << rowind[k] + 1 << " " << j + 1 << " " << values[k] << "\n";
  }
  if (!out) throw MmError{SSSVD_E_IO, "write_matrix_market: write failed for " + path};
}

template <typename F>
sssvd_status host_guarded(F&& body) {
  try {
    body();
    return SSSVD_OK;
  } catch (const MmError& e) {
    g_host_error = e.what;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_host_error = "out of host memory";
    return SSSVD_E_OOM;
  } catch (const std::exception& e) {
    g_host_error = e.what();
    return SSSVD_E_INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

sssvd_status sssvd_mm_read(const char* path, sssvd_mm_matrix** out) {
  return host_guarded([&]() {
    if (!path || !out) throw MmError{SSSVD_E_INVALID_ARGUMENT, "sssvd_mm_read: null argument"};
    *out = read_mm(path);
  });
}

void sssvd_mm_info_get(const sssvd_mm_matrix* mm, sssvd_mm_info* info) {
  info->rows = mm->rows;
  info->cols = mm->cols;
  info->nnz = (int64_t)mm->values.size();
  info->sparse = mm->sparse ? 1 : 0;
}

const double* sssvd_mm_values(const sssvd_mm_matrix* mm) { return mm->values.data(); }
const int64_t* sssvd_mm_colptr(const sssvd_mm_matrix* mm) { return mm->sparse ? mm->colptr.data() : nullptr; }
const int64_t* sssvd_mm_rowind(const sssvd_mm_matrix* mm) { return mm->sparse ? mm->rowind.data() : nullptr; }
void sssvd_mm_free(sssvd_mm_matrix* mm) { delete mm; }

sssvd_status sssvd_mm_write(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* colptr,
                            const int64_t* rowind, const double* values, const char* comment) {
  return host_guarded([&]() {
    if (!path || rows < 0 || cols < 0 || (colptr && nnz < 0))
      throw MmError{SSSVD_E_INVALID_ARGUMENT, "sssvd_mm_write: bad argument"};
    write_mm(path, rows, cols, nnz, colptr, rowind, values, comment ? comment : "");
  });
}

const char* sssvd_host_last_error(void) { return g_host_error.c_str(); }

}  // extern "C"
