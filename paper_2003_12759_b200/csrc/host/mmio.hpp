// Matrix Market coordinate IO and the report CSV (host side of the C ABI).
// Semantics follow proj/src/matrix_market.cpp:38-142 and report.cpp:46-63.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/mpg.h"

namespace mpg {

struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };

namespace mmio {

// Host CSR with new[]-allocated arrays (handed to mpg_host_csr without a copy).
struct Csr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  std::unique_ptr<int64_t[]> rowptr, colind;
  std::unique_ptr<double[]> val;
};

// read_matrix_market (matrix_market.cpp:38-98) on an in-memory text, parsed
// by `threads` host threads (0: all); errors name `origin` and the line.
Csr read(const char* data, size_t len, const std::string& origin, int threads);
Csr read_file(const std::string& path, int threads);
// write_matrix_market (matrix_market.cpp:100-142): general storage,
// row-major, shortest round-trip values; dense blocks store every entry.
std::string write(const Csr& a, int threads);
std::string write_dense(int64_t rows, int64_t cols, const double* colmajor);
void write_file(const std::string& path, const std::string& text);
// ReductionReport::write_csv (report.cpp:46-63).
std::string report_csv(const mpg_report_row* rows, int n);

}  // namespace mmio
}  // namespace mpg
