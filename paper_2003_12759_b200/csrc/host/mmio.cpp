// Matrix Market coordinate IO (proj/src/matrix_market.cpp) and the report CSV
// (proj/src/report.cpp), host side.
//
// The reference reads line by line through istringstream on one thread. Here
// the file is read into memory once and the entry section is parsed by T host
// threads: pass 1 counts lines and non-blank lines per chunk (chunks end at
// newlines), a prefix sum gives every line its file line number and entry
// index, pass 2 parses entries straight into their slots; the first error in
// file order is the one reported, and lines after the nnz-th entry are never
// looked at, exactly as the sequential reader behaves. The CSR is assembled by
// a counting sort over rows and a per-row sort + duplicate sum (the
// from_triplets rule, sparse.cpp:80-115: sorted, duplicates summed, zero sums
// kept), also across threads.
#include "mmio.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <thread>

namespace mpg {
namespace mmio {
namespace {

[[noreturn]] void fail(const std::string& origin, long line, const std::string& what) {
  throw IoError(origin + ":" + std::to_string(line) + ": " + what);
}

std::string lower(std::string s) {
  for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// Blank as the reference defines it: only ' ', '\t', '\r' (find_first_not_of(" \t\r")).
bool blank(const char* b, const char* e) {
  for (const char* p = b; p < e; ++p)
    if (*p != ' ' && *p != '\t' && *p != '\r') return false;
  return true;
}

template <class T>
bool next_num(const char*& p, const char* e, T& out) {
  while (p < e && is_ws(*p)) ++p;
  if (p == e) return false;
  const char* q = p;
  if constexpr (std::is_floating_point_v<T>) {
    // istream >> double: optional sign, digits / '.', exponent; no inf / nan words
    const char* r = q;
    if (r < e && (*r == '+' || *r == '-')) ++r;
    if (r == e || !(std::isdigit(static_cast<unsigned char>(*r)) || *r == '.')) return false;
    if (*q == '+') ++q;
  } else {
    if (q < e && *q == '+') ++q;
  }
  const auto res = std::from_chars(q, e, out);
  if (res.ec != std::errc()) return false;
  p = res.ptr;
  return true;
}

int nthreads(int t) {
  const int hw = int(std::max(1u, std::thread::hardware_concurrency()));
  return t <= 0 ? hw : std::min(t, 256);
}

template <class F>
void parallel(int T, F&& f) {
  if (T == 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(f, t);
  for (auto& x : th) x.join();
}

}  // namespace

Csr read(const char* data, size_t len, const std::string& origin, int threads) {
  const char* p = data;
  const char* end = data + len;
  long lineno = 0;
  auto getline = [&](const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    ++lineno;
    return true;
  };
  const char *b, *e;
  // header (matrix_market.cpp:42-60)
  if (!getline(b, e)) fail(origin, 1, "empty input");
  bool symmetric = false;
  {
    std::istringstream head(std::string(b, e));
    std::string banner, object, format, field, symmetry;
    head >> banner >> object >> format >> field >> symmetry;
    if (lower(banner) != "%%matrixmarket" || lower(object) != "matrix")
      fail(origin, lineno, "expected '%%MatrixMarket matrix ...' header");
    if (lower(format) != "coordinate") fail(origin, lineno, "only coordinate format is supported");
    if (lower(field) != "real") fail(origin, lineno, "only real-valued matrices are supported");
    const std::string sym = lower(symmetry);
    if (sym != "general" && sym != "symmetric") fail(origin, lineno, "symmetry must be 'general' or 'symmetric'");
    symmetric = sym == "symmetric";
  }
  // size line (:64-74)
  int64_t nrows = 0, ncols = 0, nnz = 0;
  while (true) {
    if (!getline(b, e)) fail(origin, lineno + 1, "missing size line");
    if (b < e && *b == '%') continue;
    if (blank(b, e)) continue;
    std::istringstream sz(std::string(b, e));
    if (!(sz >> nrows >> ncols >> nnz) || nrows < 0 || ncols < 0 || nnz < 0)
      fail(origin, lineno, "malformed size line (want 'rows cols nnz')");
    break;
  }
  // entries (:76-95), in parallel
  const long line0 = lineno;  // lines consumed so far
  const char* body = p;
  const size_t blen = size_t(end - body);
  const int T = int(std::max<size_t>(1, std::min<size_t>(size_t(nthreads(threads)), blen / (1 << 16) + 1)));
  std::vector<const char*> cb(size_t(T) + 1);
  cb[0] = body;
  cb[size_t(T)] = end;
  for (int t = 1; t < T; ++t) {
    const char* s = body + blen * size_t(t) / size_t(T);
    s = std::max(s, cb[size_t(t) - 1]);
    const char* nl = static_cast<const char*>(std::memchr(s, '\n', size_t(end - s)));
    cb[size_t(t)] = nl ? nl + 1 : end;
  }
  std::vector<long> lines(size_t(T), 0), ents(size_t(T), 0);
  parallel(T, [&](int t) {
    long l = 0, en = 0;
    for (const char* q = cb[size_t(t)]; q < cb[size_t(t) + 1];) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(cb[size_t(t) + 1] - q)));
      const char* le = nl ? nl : cb[size_t(t) + 1];
      ++l;
      if (!blank(q, le)) ++en;
      q = nl ? nl + 1 : cb[size_t(t) + 1];
    }
    lines[size_t(t)] = l;
    ents[size_t(t)] = en;
  });
  std::vector<long> line_off(size_t(T) + 1, 0), ent_off(size_t(T) + 1, 0);
  for (int t = 0; t < T; ++t) {
    line_off[size_t(t) + 1] = line_off[size_t(t)] + lines[size_t(t)];
    ent_off[size_t(t) + 1] = ent_off[size_t(t)] + ents[size_t(t)];
  }
  const int64_t mult = symmetric ? 2 : 1;
  // uninitialised buffers: the parsing threads first-touch their own slots
  std::unique_ptr<int64_t[]> ri(new int64_t[size_t(std::max<int64_t>(1, nnz * mult))]);
  std::unique_ptr<int64_t[]> ci(new int64_t[size_t(std::max<int64_t>(1, nnz * mult))]);
  std::unique_ptr<double[]> vv(new double[size_t(std::max<int64_t>(1, nnz * mult))]);
  std::unique_ptr<char[]> twin(new char[symmetric ? size_t(std::max<int64_t>(1, nnz)) : 1]);
  struct Err { long line = -1; std::string what; };
  std::vector<Err> errs(static_cast<size_t>(T));
  std::vector<char> ordered(static_cast<size_t>(T), 1);  // entries strictly increasing in (row, col)
  parallel(T, [&](int t) {
    long ln = line0 + line_off[size_t(t)], en = ent_off[size_t(t)];
    if (en >= nnz) return;
    int64_t pr = -1, pc = -1;
    for (const char* q = cb[size_t(t)]; q < cb[size_t(t) + 1] && en < nnz;) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(cb[size_t(t) + 1] - q)));
      const char* le = nl ? nl : cb[size_t(t) + 1];
      ++ln;
      if (!blank(q, le)) {
        const char* r = q;
        int64_t i = 0, j = 0;
        double v = 0.0;
        if (!next_num(r, le, i) || !next_num(r, le, j) || !next_num(r, le, v)) {
          errs[size_t(t)] = {ln, "malformed entry (want 'row col value')"};
          return;
        }
        if (i < 1 || i > nrows || j < 1 || j > ncols) {
          errs[size_t(t)] = {ln, "entry index out of range"};
          return;
        }
        if (i - 1 < pr || (i - 1 == pr && j - 1 <= pc)) ordered[size_t(t)] = 0;
        pr = i - 1;
        pc = j - 1;
        ri[size_t(en)] = i - 1;
        ci[size_t(en)] = j - 1;
        vv[size_t(en)] = v;
        if (symmetric) twin[size_t(en)] = i != j;
        ++en;
      }
      q = nl ? nl + 1 : cb[size_t(t) + 1];
    }
  });
  for (int t = 0; t < T; ++t)
    if (errs[size_t(t)].line >= 0) fail(origin, errs[size_t(t)].line, errs[size_t(t)].what);
  const long total = ent_off[size_t(T)];
  if (total < nnz) {
    // the reference's getline fails after the last line (:81-84)
    const long last = line0 + line_off[size_t(T)];
    fail(origin, last + 1,
         "unexpected end of file after " + std::to_string(total) + " of " + std::to_string(nnz) + " entries");
  }
  Csr out;
  out.nrows = nrows;
  out.ncols = ncols;
  out.rowptr.reset(new int64_t[size_t(nrows) + 1]);
  const int TR = std::max(1, std::min<int>(nthreads(threads), int(nrows / 4096) + 1));
  bool sorted = !symmetric;
  for (int t = 0; t < T && sorted; ++t) {
    sorted = ordered[size_t(t)] != 0;
    const int64_t k = ent_off[size_t(t)];  // first entry of chunk t vs the last of the previous ones
    if (sorted && t > 0 && k > 0 && k < nnz)
      sorted = ri[size_t(k) - 1] < ri[size_t(k)] || (ri[size_t(k) - 1] == ri[size_t(k)] && ci[size_t(k) - 1] < ci[size_t(k)]);
  }
  if (sorted) {
    // Row-major without duplicates (every file this library writes): the
    // parsed arrays are the CSR; row offsets by binary search per row.
    out.nnz = nnz;
    const int64_t* rp = ri.get();
    parallel(TR, [&](int t) {
      const int64_t r0 = (nrows + 1) * t / TR, r1 = (nrows + 1) * (t + 1) / TR;
      for (int64_t r = r0; r < r1; ++r) out.rowptr[size_t(r)] = std::lower_bound(rp, rp + nnz, r) - rp;
    });
    out.colind = std::move(ci);
    out.val = std::move(vv);
    return out;
  }
  // symmetric: mirrored entries appended
  int64_t m = nnz;
  if (symmetric)
    for (int64_t k = 0; k < nnz; ++k)
      if (twin[size_t(k)]) {
        ri[size_t(m)] = ci[size_t(k)];
        ci[size_t(m)] = ri[size_t(k)];
        vv[size_t(m)] = vv[size_t(k)];
        ++m;
      }
  // from_triplets: counting sort by row (stable), per-row sort by column, duplicates summed
  std::vector<int64_t> cnt(size_t(nrows) + 1, 0);
  for (int64_t k = 0; k < m; ++k) ++cnt[size_t(ri[size_t(k)]) + 1];
  for (int64_t r = 0; r < nrows; ++r) cnt[size_t(r) + 1] += cnt[size_t(r)];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  std::unique_ptr<std::pair<int64_t, double>[]> ent(new std::pair<int64_t, double>[size_t(std::max<int64_t>(1, m))]);
  for (int64_t k = 0; k < m; ++k) {
    const int64_t r = ri[size_t(k)];
    ent[size_t(pos[size_t(r)]++)] = {ci[size_t(k)], vv[size_t(k)]};
  }
  std::vector<int64_t> kept(size_t(nrows), 0);
  parallel(TR, [&](int t) {
    const int64_t r0 = nrows * t / TR, r1 = nrows * (t + 1) / TR;
    for (int64_t r = r0; r < r1; ++r) {
      auto* a = ent.get() + cnt[size_t(r)];
      auto* z = ent.get() + cnt[size_t(r) + 1];
      std::stable_sort(a, z, [](const auto& x, const auto& y) { return x.first < y.first; });
      int64_t w = 0;
      for (auto* q = a; q < z;) {
        const int64_t c = q->first;
        double s = 0.0;
        while (q < z && q->first == c) s += (q++)->second;
        a[w++] = {c, s};
      }
      kept[size_t(r)] = w;
    }
  });
  out.rowptr[0] = 0;
  for (int64_t r = 0; r < nrows; ++r) out.rowptr[size_t(r) + 1] = out.rowptr[size_t(r)] + kept[size_t(r)];
  out.nnz = out.rowptr[size_t(nrows)];
  out.colind.reset(new int64_t[size_t(std::max<int64_t>(1, out.nnz))]);
  out.val.reset(new double[size_t(std::max<int64_t>(1, out.nnz))]);
  parallel(TR, [&](int t) {
    const int64_t r0 = nrows * t / TR, r1 = nrows * (t + 1) / TR;
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t k = 0; k < kept[size_t(r)]; ++k) {
        out.colind[size_t(out.rowptr[size_t(r)] + k)] = ent[size_t(cnt[size_t(r)] + k)].first;
        out.val[size_t(out.rowptr[size_t(r)] + k)] = ent[size_t(cnt[size_t(r)] + k)].second;
      }
  });
  return out;
}

Csr read_file(const std::string& path, int threads) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open '" + path + "' for reading");
  std::string buf;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (sz > 0) {
    buf.resize(size_t(sz));
    const size_t got = std::fread(buf.data(), 1, size_t(sz), f);
    buf.resize(got);
  }
  std::fclose(f);
  return read(buf.data(), buf.size(), path, threads);
}

namespace {

void put_double(std::string& out, double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, size_t(res.ptr - buf));
}

void put_int(std::string& out, int64_t v) {
  char buf[32];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, size_t(res.ptr - buf));
}

}  // namespace

std::string write(const Csr& a, int threads) {
  std::string head = "%%MatrixMarket matrix coordinate real general\n";
  put_int(head, a.nrows);
  head += ' ';
  put_int(head, a.ncols);
  head += ' ';
  put_int(head, a.nnz);
  head += '\n';
  const int T = std::max(1, std::min<int>(nthreads(threads), int(a.nrows / 4096) + 1));
  std::vector<std::string> parts(static_cast<size_t>(T));
  parallel(T, [&](int t) {
    const int64_t r0 = a.nrows * t / T, r1 = a.nrows * (t + 1) / T;
    std::string& s = parts[size_t(t)];
    s.reserve(size_t(a.rowptr[size_t(r1)] - a.rowptr[size_t(r0)]) * 32);
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t k = a.rowptr[size_t(i)]; k < a.rowptr[size_t(i) + 1]; ++k) {
        put_int(s, i + 1);
        s += ' ';
        put_int(s, a.colind[size_t(k)] + 1);
        s += ' ';
        put_double(s, a.val[size_t(k)]);
        s += '\n';
      }
  });
  size_t total = head.size();
  for (auto& s : parts) total += s.size();
  std::string out;
  out.reserve(total);
  out += head;
  for (auto& s : parts) out += s;
  return out;
}

std::string write_dense(int64_t rows, int64_t cols, const double* m) {
  std::string out = "%%MatrixMarket matrix coordinate real general\n";
  put_int(out, rows);
  out += ' ';
  put_int(out, cols);
  out += ' ';
  put_int(out, rows * cols);
  out += '\n';
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      put_int(out, i + 1);
      out += ' ';
      put_int(out, j + 1);
      out += ' ';
      put_double(out, m[i + rows * j]);
      out += '\n';
    }
  return out;
}

void write_file(const std::string& path, const std::string& text) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError("cannot open '" + path + "' for writing");
  const size_t put = std::fwrite(text.data(), 1, text.size(), f);
  const int cl = std::fclose(f);
  if (put != text.size() || cl != 0) throw IoError("write to '" + path + "' failed");
}

std::string report_csv(const mpg_report_row* rows, int n) {
  static const char* const kinds[] = {"none", "fresh", "horizontal", "vertical", "reused_same_matrix"};
  std::ostringstream os;  // default ostream formatting, as report.cpp:46-63
  auto metric = [&](double v) {
    os << ',';
    if (!std::isnan(v)) os << v;
  };
  os << "sweep,point,precond,solves,precond_build_seconds,gmres_iterations,"
        "gmres_seconds,min_residual,matrix_change,standard_residual,"
        "first_approach_min_residual\n";
  int solves = 0;
  double build = 0.0, secs = 0.0;
  long its = 0;
  for (int k = 0; k < n; ++k) {
    const mpg_report_row& r = rows[k];
    os << r.sweep << ',' << r.point << ',' << (r.kind >= 0 && r.kind < 5 ? kinds[r.kind] : "unknown") << ','
       << r.solves << ',' << r.build_seconds << ',' << long(r.iterations) << ',' << r.gmres_seconds;
    metric(r.min_residual);
    metric(r.matrix_change);
    metric(r.standard_residual);
    metric(std::nan(""));  // first_approach_min_residual: not produced on this path
    os << '\n';
    solves += r.solves;
    build += r.build_seconds;
    its += long(r.iterations);
    secs += r.gmres_seconds;
  }
  os << "TOTAL,," << ',' << solves << ',' << build << ',' << its << ',' << secs << ",,,,\n";
  return os.str();
}

}  // namespace mmio
}  // namespace mpg
