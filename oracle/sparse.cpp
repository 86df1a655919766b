// CPU ORACLE — test infrastructure only (see oracle.hpp).
// Restates proj/src/sparse.cpp (CSR + CSC shadow, SpMV, transpose, column
// submatrix extraction, linear combination) and proj/src/kron.cpp (N = 0
// Kronecker operator, generalised with a mass matrix E).
#include <algorithm>
#include <cmath>
#include <string>

#include "oracle.hpp"

namespace oracle {

// proj/src/sparse.cpp:27-46
void Csr::build_shadow() {
  const index_t nnz = index_t(colind.size());
  colptr.assign(static_cast<size_t>(ncols) + 1, 0);
  for (index_t k = 0; k < nnz; ++k) ++colptr[size_t(colind[size_t(k)]) + 1];
  for (index_t j = 0; j < ncols; ++j) colptr[size_t(j) + 1] += colptr[size_t(j)];
  srow.resize(static_cast<size_t>(nnz));
  sval.resize(static_cast<size_t>(nnz));
  std::vector<index_t> cursor(colptr.begin(), colptr.end() - 1);
  for (index_t i = 0; i < nrows; ++i)
    for (index_t k = rowptr[size_t(i)]; k < rowptr[size_t(i) + 1]; ++k) {
      const index_t slot = cursor[size_t(colind[size_t(k)])]++;
      srow[size_t(slot)] = i;
      sval[size_t(slot)] = val[size_t(k)];
    }
}

// proj/src/sparse.cpp:48-74
void Csr::validate() const {
  if (nrows < 0 || ncols < 0) throw std::invalid_argument("sparse: negative dimension");
  if (rowptr.size() != size_t(nrows) + 1) throw std::invalid_argument("sparse: row_offsets length must be nrows + 1");
  if (rowptr.front() != 0) throw std::invalid_argument("sparse: row_offsets must start at 0");
  if (colind.size() != val.size()) throw std::invalid_argument("sparse: col_indices and values lengths differ");
  if (rowptr.back() != index_t(colind.size())) throw std::invalid_argument("sparse: row_offsets must end at nnz");
  for (index_t i = 0; i < nrows; ++i) {
    const index_t lo = rowptr[size_t(i)], hi = rowptr[size_t(i) + 1];
    if (hi < lo) throw std::invalid_argument("sparse: row_offsets must be nondecreasing");
    index_t prev = -1;
    for (index_t k = lo; k < hi; ++k) {
      const index_t j = colind[size_t(k)];
      if (j < 0 || j >= ncols) throw std::invalid_argument("sparse: column index out of range in row " + std::to_string(i));
      if (j <= prev) throw std::invalid_argument("sparse: column indices must be strictly increasing in row " + std::to_string(i));
      prev = j;
    }
  }
}

// proj/src/sparse.cpp:80-115 (duplicates summed; exact-zero sums kept)
Csr Csr::from_triplets(index_t nr, index_t nc, std::vector<Triplet> t) {
  if (nr < 0 || nc < 0) throw std::invalid_argument("sparse: negative dimension");
  for (const Triplet& x : t)
    if (x.row < 0 || x.row >= nr || x.col < 0 || x.col >= nc)
      throw std::invalid_argument("sparse: triplet index out of range");
  std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  Csr m;
  m.nrows = nr;
  m.ncols = nc;
  m.rowptr.assign(static_cast<size_t>(nr) + 1, 0);
  m.colind.reserve(t.size());
  m.val.reserve(t.size());
  size_t p = 0;
  while (p < t.size()) {
    const index_t r = t[p].row, c = t[p].col;
    double sum = 0.0;
    while (p < t.size() && t[p].row == r && t[p].col == c) sum += t[p++].value;
    m.colind.push_back(c);
    m.val.push_back(sum);
    ++m.rowptr[size_t(r) + 1];
  }
  for (index_t i = 0; i < nr; ++i) m.rowptr[size_t(i) + 1] += m.rowptr[size_t(i)];
  m.build_shadow();
  return m;
}

Csr Csr::from_csr(index_t nr, index_t nc, std::vector<index_t> rp, std::vector<index_t> ci, std::vector<double> v) {
  Csr m;
  m.nrows = nr;
  m.ncols = nc;
  m.rowptr = std::move(rp);
  m.colind = std::move(ci);
  m.val = std::move(v);
  m.validate();
  m.build_shadow();
  return m;
}

Csr Csr::identity(index_t n) {
  std::vector<Triplet> t;
  for (index_t i = 0; i < n; ++i) t.push_back({i, i, 1.0});
  return from_triplets(n, n, t);
}

Csr Csr::diagonal(const Vec& d) {
  std::vector<Triplet> t;
  for (size_t i = 0; i < d.size(); ++i) t.push_back({index_t(i), index_t(i), d[i]});
  return from_triplets(index_t(d.size()), index_t(d.size()), t);
}

Csr Csr::zero(index_t nr, index_t nc) {
  Csr m;
  m.nrows = nr;
  m.ncols = nc;
  m.rowptr.assign(static_cast<size_t>(nr) + 1, 0);
  m.build_shadow();
  return m;
}

// proj/src/sparse.cpp:156-202 (cancelled entries dropped)
Csr Csr::linear_combination(const std::vector<std::pair<double, const Csr*>>& terms) {
  if (terms.empty()) throw std::invalid_argument("linear_combination: no terms");
  const index_t nr = terms.front().second->nrows, nc = terms.front().second->ncols;
  for (const auto& t : terms)
    if (t.second->nrows != nr || t.second->ncols != nc) throw std::invalid_argument("linear_combination: dimension mismatch");
  Csr m;
  m.nrows = nr;
  m.ncols = nc;
  m.rowptr.assign(static_cast<size_t>(nr) + 1, 0);
  std::vector<std::pair<index_t, double>> merged;
  for (index_t i = 0; i < nr; ++i) {
    merged.clear();
    for (const auto& [coeff, mat] : terms)
      for (index_t k = mat->rowptr[size_t(i)]; k < mat->rowptr[size_t(i) + 1]; ++k)
        merged.emplace_back(mat->colind[size_t(k)], coeff * mat->val[size_t(k)]);
    std::stable_sort(merged.begin(), merged.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    size_t p = 0;
    while (p < merged.size()) {
      const index_t j = merged[p].first;
      double sum = 0.0;
      while (p < merged.size() && merged[p].first == j) sum += merged[p++].second;
      if (sum != 0.0) {
        m.colind.push_back(j);
        m.val.push_back(sum);
        ++m.rowptr[size_t(i) + 1];
      }
    }
  }
  for (index_t i = 0; i < nr; ++i) m.rowptr[size_t(i) + 1] += m.rowptr[size_t(i)];
  m.build_shadow();
  return m;
}

// proj/src/sparse.cpp:236-249 (fixed per-row order)
void Csr::multiply(const Vec& x, Vec& y) const {
  if (index_t(x.size()) != ncols) throw std::invalid_argument("sparse multiply: dimension mismatch");
  y.resize(static_cast<size_t>(nrows));
  for (index_t i = 0; i < nrows; ++i) {
    double acc = 0.0;
    for (index_t k = rowptr[size_t(i)]; k < rowptr[size_t(i) + 1]; ++k) acc += val[size_t(k)] * x[size_t(colind[size_t(k)])];
    y[size_t(i)] = acc;
  }
}

// proj/src/sparse.cpp:257-269
Vec Csr::multiply_transpose(const Vec& x) const {
  if (index_t(x.size()) != nrows) throw std::invalid_argument("sparse multiply_transpose: dimension mismatch");
  Vec y(static_cast<size_t>(ncols));
  for (index_t j = 0; j < ncols; ++j) {
    double acc = 0.0;
    for (index_t k = colptr[size_t(j)]; k < colptr[size_t(j) + 1]; ++k) acc += sval[size_t(k)] * x[size_t(srow[size_t(k)])];
    y[size_t(j)] = acc;
  }
  return y;
}

Dense Csr::multiply(const Dense& x) const {
  if (x.rows != ncols) throw std::invalid_argument("sparse multiply: dimension mismatch");
  Dense y(nrows, x.cols);
  Vec in(static_cast<size_t>(ncols)), out;
  for (index_t c = 0; c < x.cols; ++c) {
    std::copy(x.col(c), x.col(c) + ncols, in.begin());
    multiply(in, out);
    std::copy(out.begin(), out.end(), y.col(c));
  }
  return y;
}

// proj/src/sparse.cpp:289-299
Csr Csr::transpose() const {
  Csr t;
  t.nrows = ncols;
  t.ncols = nrows;
  t.rowptr = colptr;
  t.colind = srow;
  t.val = sval;
  t.build_shadow();
  return t;
}

double Csr::frobenius_norm() const {
  double s = 0.0;
  for (double v : val) s += v * v;
  return std::sqrt(s);
}

Dense Csr::to_dense() const {
  if (nrows * ncols > (index_t(1) << 26)) throw std::invalid_argument("sparse to_dense: matrix too large to materialize");
  Dense d(nrows, ncols);
  for (index_t i = 0; i < nrows; ++i)
    for (index_t k = rowptr[size_t(i)]; k < rowptr[size_t(i) + 1]; ++k) d(i, colind[size_t(k)]) = val[size_t(k)];
  return d;
}

// proj/src/sparse.cpp:313-345
Csr::ColumnSubmatrix Csr::extract_column_submatrix(const std::vector<index_t>& pattern) const {
  if (pattern.empty()) throw std::invalid_argument("extract_column_submatrix: empty pattern");
  for (index_t j : pattern)
    if (j < 0 || j >= ncols) throw std::invalid_argument("extract_column_submatrix: column index out of range");
  ColumnSubmatrix out;
  for (index_t j : pattern)
    for (index_t k = colptr[size_t(j)]; k < colptr[size_t(j) + 1]; ++k) out.row_map.push_back(srow[size_t(k)]);
  std::sort(out.row_map.begin(), out.row_map.end());
  out.row_map.erase(std::unique(out.row_map.begin(), out.row_map.end()), out.row_map.end());
  std::vector<index_t> seen(pattern);
  std::sort(seen.begin(), seen.end());
  if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
    throw std::invalid_argument("extract_column_submatrix: repeated pattern index");
  out.block = Dense(index_t(out.row_map.size()), index_t(pattern.size()));
  for (size_t c = 0; c < pattern.size(); ++c)
    for (index_t k = colptr[size_t(pattern[c])]; k < colptr[size_t(pattern[c]) + 1]; ++k) {
      const auto it = std::lower_bound(out.row_map.begin(), out.row_map.end(), srow[size_t(k)]);
      out.block(index_t(it - out.row_map.begin()), index_t(c)) = sval[size_t(k)];
    }
  return out;
}

double frobenius_distance(const Csr& a, const Csr& b) {
  return Csr::linear_combination({{1.0, &a}, {-1.0, &b}}).frobenius_norm();
}

// proj/src/kron.cpp:34-64 with coupler-free operator, generalised:
// vec(-E X Lambda^T - A X); E = I reproduces the reference exactly.
void KronOp::apply(const Vec& in, Vec& out) const {
  const index_t n = a->nrows, r = lambda.rows;
  if (index_t(in.size()) != n * r) throw std::invalid_argument("kronecker apply: dimension mismatch");
  out.assign(static_cast<size_t>(n * r), 0.0);
  Vec ex(static_cast<size_t>(n * r));
  Vec col(static_cast<size_t>(n)), tmp;
  for (index_t c = 0; c < r; ++c) {
    if (e) {
      std::copy(in.begin() + c * n, in.begin() + (c + 1) * n, col.begin());
      e->multiply(col, tmp);
      std::copy(tmp.begin(), tmp.end(), ex.begin() + c * n);
    } else {
      std::copy(in.begin() + c * n, in.begin() + (c + 1) * n, ex.begin() + c * n);
    }
  }
  // y = -(E X) Lambda^T
  for (index_t c = 0; c < r; ++c)
    for (index_t k = 0; k < r; ++k) {
      const double l = lambda(c, k);
      if (l == 0.0) continue;
      for (index_t i = 0; i < n; ++i) out[size_t(c * n + i)] -= l * ex[size_t(k * n + i)];
    }
  for (index_t c = 0; c < r; ++c) {
    std::copy(in.begin() + c * n, in.begin() + (c + 1) * n, col.begin());
    a->multiply(col, tmp);
    for (index_t i = 0; i < n; ++i) out[size_t(c * n + i)] -= tmp[size_t(i)];
  }
  // couplers: mixed = X S (n x r), y(:, c) -= N mixed(:, c)  (kron.cpp:54-63)
  for (const Coupler& cp : couplers) {
    for (index_t c = 0; c < r; ++c) {
      std::fill(col.begin(), col.end(), 0.0);
      for (index_t b = 0; b < r; ++b) {
        const double sv = cp.small(b, c);
        if (sv == 0.0) continue;
        for (index_t i = 0; i < n; ++i) col[size_t(i)] += in[size_t(b * n + i)] * sv;
      }
      cp.sparse->multiply(col, tmp);
      for (index_t i = 0; i < n; ++i) out[size_t(c * n + i)] -= tmp[size_t(i)];
    }
  }
}

// proj/src/kron.cpp:72-131 (cap estimate counts Lambda entries times nnz(E))
Csr assemble_explicit(const KronOp& op, index_t max_nnz) {
  const index_t n = op.a->nrows, r = op.lambda.rows;
  index_t lambda_nnz = 0;
  for (index_t i = 0; i < r; ++i)
    for (index_t j = 0; j < r; ++j) lambda_nnz += op.lambda(i, j) != 0.0;
  const index_t e_nnz = op.e ? op.e->nnz() : n;
  index_t estimate = lambda_nnz * e_nnz + r * op.a->nnz();
  for (const auto& cp : op.couplers) {
    index_t small_nnz = 0;
    for (index_t i = 0; i < r; ++i)
      for (index_t j = 0; j < r; ++j) small_nnz += cp.small(i, j) != 0.0;
    estimate += small_nnz * cp.sparse->nnz();
  }
  if (estimate > max_nnz)
    throw ConfigError("explicit operator assembly needs about " + std::to_string(estimate) +
                      " entries, above the cap of " + std::to_string(max_nnz) +
                      "; rerun with a fresh approximate inverse per sweep or without preconditioning");
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(estimate));
  for (index_t bi = 0; bi < r; ++bi)
    for (index_t bj = 0; bj < r; ++bj) {
      const double v = op.lambda(bi, bj);
      if (v == 0.0) continue;
      if (op.e) {
        for (index_t i = 0; i < n; ++i)
          for (index_t k = op.e->rowptr[size_t(i)]; k < op.e->rowptr[size_t(i) + 1]; ++k)
            t.push_back({bi * n + i, bj * n + op.e->colind[size_t(k)], -v * op.e->val[size_t(k)]});
      } else {
        for (index_t i = 0; i < n; ++i) t.push_back({bi * n + i, bj * n + i, -v});
      }
    }
  for (index_t b = 0; b < r; ++b)
    for (index_t i = 0; i < n; ++i)
      for (index_t k = op.a->rowptr[size_t(i)]; k < op.a->rowptr[size_t(i) + 1]; ++k)
        t.push_back({b * n + i, b * n + op.a->colind[size_t(k)], -op.a->val[size_t(k)]});
  // -(S^T (x) N): block (bi, bj) is -S(bj, bi) N  (kron.cpp:115-128)
  for (const auto& cp : op.couplers)
    for (index_t bi = 0; bi < r; ++bi)
      for (index_t bj = 0; bj < r; ++bj) {
        const double sv = cp.small(bj, bi);
        if (sv == 0.0) continue;
        const Csr& nm = *cp.sparse;
        for (index_t i = 0; i < n; ++i)
          for (index_t k = nm.rowptr[size_t(i)]; k < nm.rowptr[size_t(i) + 1]; ++k)
            t.push_back({bi * n + i, bj * n + nm.colind[size_t(k)], -sv * nm.val[size_t(k)]});
      }
  return Csr::from_triplets(n * r, n * r, std::move(t));
}

}  // namespace oracle
