// CPU ORACLE -- test infrastructure only. A C entry point over the reference's
// own Eigen-free sources, compiled unchanged from /root/reference by
// oracle/ref/Makefile into oracle/_ref/libref_report.so (never shipped, never
// linked by the product): ReductionReport::write_csv (proj/src/report.cpp:46-63),
// parallel_for (proj/src/parallel.cpp:13-46) and shortest (format.hpp:12-16).
// tests/test_ref_report.py diffs libmpg's mpg_report_csv and the oracle
// against them byte for byte.
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "morprec/format.hpp"
#include "morprec/parallel.hpp"
#include "morprec/report.hpp"

extern "C" {

// rows: the mpg_report_row layout (include/mpg.h).
typedef struct {
  int sweep, point, kind, solves;
  long long iterations;
  double build_seconds, gmres_seconds, min_residual, matrix_change, standard_residual;
} ref_row;

static char* dup(const std::string& s, long long* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  *len = static_cast<long long>(s.size());
  return p;
}

char* ref_report_csv(const ref_row* rows, int n, long long* len) {
  morprec::ReductionReport rep;
  for (int i = 0; i < n; ++i) {
    morprec::ReportRow r;
    r.sweep = rows[i].sweep;
    r.point = rows[i].point;
    r.kind = static_cast<morprec::PrecondKind>(rows[i].kind);
    r.solves = rows[i].solves;
    r.precond_build_seconds = rows[i].build_seconds;
    r.gmres_iterations = static_cast<long>(rows[i].iterations);
    r.gmres_seconds = rows[i].gmres_seconds;
    r.min_residual = rows[i].min_residual;
    r.matrix_change = rows[i].matrix_change;
    r.standard_residual = rows[i].standard_residual;
    rep.rows.push_back(r);
  }
  std::ostringstream os;
  rep.write_csv(os);
  return dup(os.str(), len);
}

char* ref_shortest(double v, long long* len) { return dup(morprec::shortest(v), len); }

// parallel_for over [0, n) with `threads`: out[i] = i * i (covers the chunking).
void ref_parallel_squares(long long n, int threads, long long* out) {
  morprec::parallel_for(0, static_cast<std::int64_t>(n), threads,
                        [out](std::int64_t i) { out[i] = static_cast<long long>(i) * static_cast<long long>(i); });
}

void ref_free(char* p) { std::free(p); }
}
