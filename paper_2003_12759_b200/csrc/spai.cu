// K4: sparse approximate inverse and update-factor builds, one warp per column
// (spai_build, proj/src/spai.cpp:175-238; update_build, proj/src/chain.cpp:16-98;
// the shared adaptive column loop, spai.cpp:89-154; solve_pattern,
// spai.cpp:16-41; initial_pattern, spai.cpp:43-87).
//
// Per column the warp builds the pattern J (sorted), the touched rows I
// (sorted union of rows of A(:, J)), gathers the dense block A(I, J) and solves
// the least-squares problem with a Householder QR with column pivoting that
// follows Eigen's ColPivHouseholderQR (pivot = largest updated column norm,
// first index on ties; norm downdating with recomputation below sqrt(eps);
// rank = #|R_ii| > max|R_jj| * min(m, p) * eps). Augmentation picks the
// largest-magnitude residual row outside the pattern (ties to the lowest
// index), up to max_pattern_sweeps times. Rank-deficient columns fall back to
// 1/a_jj (SPAI) or the identity column (update). The result is written as the
// CSR of P^T (column lists) and transposed on the device.
//
// Lanes own rows (i = lane mod 32) of the dense block, which lives in a
// per-warp workspace in global memory (L1/L2 resident). The phase functions
// are kept out of line: inlined twice (first solve + augmentation sweeps) the
// kernel was 200 KB of SASS and stalled on instruction fetch (ncu:
// no_instructions 47 % of samples); out of line it also needs 72 instead of
// 128 registers, so more warps hide the workspace latency (C3 2.5 -> 1.7 s).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cfloat>

#include <climits>
#include <cstdio>
#include <string>

#include "runtime.cuh"

namespace mpg {
namespace {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct SpaiParams {
  CsrView at;      // CSR of A^T: column j of A = row j of A^T (sorted rows)
  CsrView prevt;   // CSR of A_prev^T (update builds), nrows == 0 for SPAI
  int n;
  int update;
  int pattern_kind;
  double fill_tol;
  int max_fill, max_sweeps;
  int PMAX, IMAX, SORTN, RHSMAX;
  // per-warp workspace strides
  size_t ws_doubles, ws_ints;
  double* wsd;
  int* wsi;
  // outputs
  int* cnt;        // per column
  int* orow;       // n * PMAX
  double* oval;    // n * PMAX
  double* ores;    // residual (SPAI) or residual^2 (update) per column
  int* ofb;        // fallback flags
  int* next;       // work counter
  const int* fixed_J;  // spai_column_solve: fixed sorted pattern for column `only_col`
  const int* ipat;     // pattern_kind 2: initial pattern of column j at ipat[j * istride], icnt[j] entries
  const int* icnt;
  int istride;
  int fixed_np, only_col, raw;
  unsigned long long* phase;  // MPG_SPAI_PHASES: clock cycles summed over warps in rows / gather / QR / residual
};

struct WarpWS {
  double* D;       // IMAX * PMAX
  double* rhsl;    // IMAX
  double* resid;   // IMAX + RHSMAX
  double* coef;    // PMAX
  double* hc;      // PMAX
  double* upd;     // PMAX
  double* dir;     // PMAX
  int* J;          // PMAX
  int* perm;       // PMAX
  int* tr;         // PMAX
  int* I;          // IMAX
  int* I2;         // IMAX
  int* sb;         // SORTN
};

__device__ int lower_bound_i(const int* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sorted unique union of the rows of A(:, J) into I; returns |I|.
__device__ __noinline__ int build_rows(const SpaiParams& P, const WarpWS& w, int np, int lane) {
  int total = 0;
  for (int c = 0; c < np; ++c) {
    const int j = w.J[c];
    const int b = P.at.rowptr[j], e = P.at.rowptr[j + 1];
    for (int k = lane; k < e - b; k += 32) w.sb[total + k] = P.at.colind[b + k];
    total += e - b;
  }
  int N = 1;
  while (N < total) N <<= 1;
  for (int i = total + lane; i < N; i += 32) w.sb[i] = INT_MAX;
  __syncwarp();
  for (int size = 2; size <= N; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < N / 2; i += 32) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const int a = w.sb[lo], b = w.sb[hi];
        if ((a > b) == asc) { w.sb[lo] = b; w.sb[hi] = a; }
      }
      __syncwarp();
    }
  int m = 0;
  for (int base = 0; base < total; base += 32) {
    const int i = base + lane;
    const bool keep = i < total && (i == 0 || w.sb[i] != w.sb[i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) w.I[m + __popc(bal & ((1u << lane) - 1u))] = w.sb[i];
    m += __popc(bal);
  }
  __syncwarp();
  return m;
}

// Dense block A(I, J) column-major (ld = m) and the restricted right-hand side.
__device__ __noinline__ void gather(const SpaiParams& P, const WarpWS& w, int np, int m, const int* rr, const double* rv, int rn,
                       double& outside_sq, int lane) {
  for (int i = lane; i < m * np; i += 32) w.D[i] = 0.0;
  for (int i = lane; i < m; i += 32) w.rhsl[i] = 0.0;
  __syncwarp();
  for (int c = 0; c < np; ++c) {
    const int j = w.J[c];
    const int b = P.at.rowptr[j], e = P.at.rowptr[j + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int pos = lower_bound_i(w.I, m, P.at.colind[k]);
      w.D[pos + size_t(c) * m] = P.at.val[k];
    }
  }
  double o = 0.0;
  for (int k = lane; k < rn; k += 32) {
    const int pos = lower_bound_i(w.I, m, rr[k]);
    if (pos < m && w.I[pos] == rr[k]) w.rhsl[pos] = rv[k];
    else o += rv[k] * rv[k];
  }
  outside_sq = wsum(o);
  __syncwarp();
}

// Householder QR with column pivoting (Eigen ColPivHouseholderQR) and solve.
// Returns rank_deficient; coefficients (in pattern order) in w.coef.
__device__ __noinline__ bool qr_solve(const WarpWS& w, int m, int p, int lane) {
  double* D = w.D;
  const int size = min(m, p);
  double maxnorm = 0.0;
  for (int c = 0; c < p; ++c) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(D[r + size_t(c) * m], D[r + size_t(c) * m], s);
    s = sqrt(wsum(s));
    if (lane == 0) { w.upd[c] = s; w.dir[c] = s; }
    maxnorm = fmax(maxnorm, s);
  }
  __syncwarp();
  const double eps = DBL_EPSILON;
  const double thr_helper = (maxnorm * eps) * (maxnorm * eps) / double(m);
  const double downdate = sqrt(eps);
  int nz = size;
  double maxpivot = 0.0;
  for (int k = 0; k < size; ++k) {
    // pivot: largest updated norm, first index on ties
    double bv = -1.0;
    int bj = p;
    for (int j = k + lane; j < p; j += 32) {
      const double v = w.upd[j];
      if (v > bv) { bv = v; bj = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
    }
    if (nz == size && bv * bv < thr_helper * double(m - k)) nz = k;
    if (lane == 0) w.tr[k] = bj;
    if (bj != k) {
      for (int r = lane; r < m; r += 32) {
        const double t = D[r + size_t(k) * m];
        D[r + size_t(k) * m] = D[r + size_t(bj) * m];
        D[r + size_t(bj) * m] = t;
      }
      if (lane == 0) {
        double t = w.upd[k]; w.upd[k] = w.upd[bj]; w.upd[bj] = t;
        t = w.dir[k]; w.dir[k] = w.dir[bj]; w.dir[bj] = t;
      }
    }
    __syncwarp();
    // Householder reflector of column k, rows k..m-1
    double* col = D + size_t(k) * m;
    double tail = 0.0;
    for (int r = k + 1 + lane; r < m; r += 32) tail = fma(col[r], col[r], tail);
    tail = wsum(tail);
    const double c0 = col[k];
    double tau, beta;
    if (tail <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      for (int r = k + 1 + lane; r < m; r += 32) col[r] = 0.0;
    } else {
      beta = sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double den = c0 - beta;
      for (int r = k + 1 + lane; r < m; r += 32) col[r] = col[r] / den;
      tau = (beta - c0) / beta;
    }
    __syncwarp();
    if (lane == 0) { col[k] = beta; w.hc[k] = tau; }
    maxpivot = fmax(maxpivot, fabs(beta));
    __syncwarp();
    // apply to the remaining columns, 4 at a time
    if (tau != 0.0) {
      for (int j0 = k + 1; j0 < p; j0 += 4) {
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        const int nj = min(4, p - j0);
        for (int r = k + 1 + lane; r < m; r += 32) {
          const double v = col[r];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nj) t[q] = fma(v, D[r + size_t(j0 + q) * m], t[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = wsum(t[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= nj) continue;
          double* cj = D + size_t(j0 + q) * m;
          const double tt = t[q] + cj[k];
          for (int r = k + 1 + lane; r < m; r += 32) cj[r] = fma(-tau * col[r], tt, cj[r]);
          __syncwarp();
          if (lane == 0) cj[k] -= tau * tt;
        }
      }
    }
    __syncwarp();
    // norm downdate
    unsigned need = 0;
    for (int j = k + 1 + lane, it = 0; j < p; j += 32, ++it) {
      const double u = w.upd[j];
      bool rec = false;
      if (u != 0.0) {
        double t = fabs(D[k + size_t(j) * m]) / u;
        t = (1.0 + t) * (1.0 - t);
        if (t < 0.0) t = 0.0;
        const double ratio = u / w.dir[j];
        const double t2 = t * ratio * ratio;
        if (t2 <= downdate) rec = true;
        else w.upd[j] = u * sqrt(t);
      }
      if (rec) need |= 1u << it;
    }
    for (int it = 0; it * 32 + k + 1 < p; ++it) {
      unsigned bal = __ballot_sync(0xffffffffu, (need >> it) & 1u);
      while (bal) {
        const int src = __ffs(bal) - 1;
        bal &= bal - 1;
        const int j = k + 1 + it * 32 + src;
        double s = 0.0;
        for (int r = k + 1 + lane; r < m; r += 32) s = fma(D[r + size_t(j) * m], D[r + size_t(j) * m], s);
        s = sqrt(wsum(s));
        if (lane == 0) { w.dir[j] = s; w.upd[j] = s; }
      }
    }
    __syncwarp();
  }
  // rank (Eigen: threshold = min(m, p) * eps relative to the largest pivot)
  int rank = 0;
  const double thr = fabs(maxpivot) * double(size) * eps;
  for (int i = 0; i < nz; ++i) rank += fabs(D[i + size_t(i) * m]) > thr;
  // solve: c = Q^T rhs over nz reflectors, then R^{-1}
  for (int kk = 0; kk < nz; ++kk) {
    const double* col = D + size_t(kk) * m;
    const double tau = w.hc[kk];
    if (tau == 0.0) continue;
    double t = 0.0;
    for (int r = kk + 1 + lane; r < m; r += 32) t = fma(col[r], w.rhsl[r], t);
    t = wsum(t) + w.rhsl[kk];
    for (int r = kk + 1 + lane; r < m; r += 32) w.rhsl[r] = fma(-tau * col[r], t, w.rhsl[r]);
    __syncwarp();
    if (lane == 0) w.rhsl[kk] -= tau * t;
    __syncwarp();
  }
  for (int i = nz - 1; i >= 0; --i) {
    double s = 0.0;
    for (int j = i + 1 + lane; j < nz; j += 32) s = fma(D[i + size_t(j) * m], w.rhsl[j], s);
    s = wsum(s);
    if (lane == 0) w.rhsl[i] = (w.rhsl[i] - s) / D[i + size_t(i) * m];
    __syncwarp();
  }
  // permutation: identity, then transpositions k <-> tr[k]
  if (lane == 0) {
    for (int i = 0; i < p; ++i) w.perm[i] = i;
    for (int k = 0; k < size; ++k) {
      const int t = w.perm[k];
      w.perm[k] = w.perm[w.tr[k]];
      w.perm[w.tr[k]] = t;
    }
  }
  __syncwarp();
  for (int i = lane; i < p; i += 32) w.coef[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < nz; i += 32) w.coef[w.perm[i]] = w.rhsl[i];
  __syncwarp();
  return rank < p;
}

// Residual over I (into w.resid[0..m)); returns ||rhs - A q||^2 on I.
__device__ __noinline__ double residual_on_I(const SpaiParams& P, const WarpWS& w, int np, int m, const int* rr, const double* rv,
                                int rn, int lane) {
  for (int i = lane; i < m; i += 32) w.resid[i] = 0.0;
  __syncwarp();
  for (int k = lane; k < rn; k += 32) {
    const int pos = lower_bound_i(w.I, m, rr[k]);
    if (pos < m && w.I[pos] == rr[k]) w.resid[pos] = rv[k];
  }
  __syncwarp();
  for (int c = 0; c < np; ++c) {
    const int j = w.J[c];
    const double q = w.coef[c];
    const int b = P.at.rowptr[j], e = P.at.rowptr[j + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int pos = lower_bound_i(w.I, m, P.at.colind[k]);
      w.resid[pos] = fma(-q, P.at.val[k], w.resid[pos]);
    }
    __syncwarp();
  }
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s = fma(w.resid[i], w.resid[i], s);
  return wsum(s);
}

// ---- PatternOfAPow initial patterns (spai.cpp:55-71) --------------------------------
// Column col's pattern is {col} and every row reachable from col in 1..k
// expansions "row i of column j" (the structural support of A e_col, ..., A^k
// e_col), sorted, truncated to the lowest max_fill indices with the diagonal
// kept (spai.cpp:74-85). One CTA per column: each expansion gathers the
// frontier's column supports into shared memory, sorts them (bitonic), keeps
// the entries not seen before as the next frontier and merges them into the
// seen set. A column whose expansion exceeds the shared-memory bounds raises
// an overflow flag (ConfigError on the host).
constexpr int AP_THREADS = 256, AP_CAND = 4096, AP_SEEN = 2048;

__device__ void ap_bitonic(int* keys, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = keys[i], b = keys[ixj];
          if ((a > b) == ((i & k) == 0)) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
    }
  __syncthreads();
}

__device__ bool ap_contains(const int* a, int n, int x) {
  const int pos = lower_bound_i(a, n, x);
  return pos < n && a[pos] == x;
}

__global__ void __launch_bounds__(AP_THREADS) k_apow_pattern(CsrView at, int power, int max_fill, int* ipat, int* icnt,
                                                              int* overflow) {
  __shared__ int cand[AP_CAND], seen[AP_SEEN], front[AP_SEEN], scan[AP_THREADS];
  __shared__ int s_nfront, s_nseen, s_total, s_bad;
  for (int col = blockIdx.x; col < at.nrows; col += gridDim.x) {
    if (threadIdx.x == 0) {
      front[0] = col;
      s_nfront = 1;
      s_nseen = 0;
      s_bad = 0;
    }
    __syncthreads();
    for (int step = 0; step < max(power, 1); ++step) {
      const int nfront = s_nfront, nseen = s_nseen;
      if (nfront == 0) break;
      // gather the frontier's column supports (rows of A(:, j) = row j of A^T)
      if (threadIdx.x == 0) {
        int t = 0;
        for (int f = 0; f < nfront; ++f) t += at.rowptr[front[f] + 1] - at.rowptr[front[f]];
        s_total = t;
      }
      __syncthreads();
      const int total = s_total;
      if (total > AP_CAND) {
        if (threadIdx.x == 0) s_bad = 1;
        __syncthreads();
        break;
      }
      if (threadIdx.x == 0) {
        int o = 0;
        for (int f = 0; f < nfront; ++f) {
          const int b = at.rowptr[front[f]], e = at.rowptr[front[f] + 1];
          for (int q = b; q < e; ++q) cand[o++] = at.colind[q];
        }
      }
      __syncthreads();
      int P = 1;
      while (P < total) P <<= 1;
      for (int i = total + threadIdx.x; i < P; i += blockDim.x) cand[i] = INT_MAX;
      ap_bitonic(cand, P);
      // unique candidates not seen before -> the next frontier
      const int per = (P + blockDim.x - 1) / blockDim.x;
      const int b = threadIdx.x * per, e = min(P, b + per);
      int c = 0;
      for (int i = b; i < e; ++i)
        if (cand[i] != INT_MAX && (i == 0 || cand[i] != cand[i - 1]) && !ap_contains(seen, nseen, cand[i])) ++c;
      scan[threadIdx.x] = c;
      __syncthreads();
      for (int off = 1; off < blockDim.x; off <<= 1) {
        const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
      }
      const int nnew = scan[blockDim.x - 1];
      if (nseen + nnew > AP_SEEN) {
        if (threadIdx.x == 0) s_bad = 1;
        __syncthreads();
        break;
      }
      int pos = scan[threadIdx.x] - c;
      for (int i = b; i < e; ++i)
        if (cand[i] != INT_MAX && (i == 0 || cand[i] != cand[i - 1]) && !ap_contains(seen, nseen, cand[i]))
          front[pos++] = cand[i];
      __syncthreads();
      // seen <- sorted(seen U front)
      for (int i = threadIdx.x; i < nnew; i += blockDim.x) cand[i] = front[i];
      for (int i = threadIdx.x; i < nseen; i += blockDim.x) cand[nnew + i] = seen[i];
      int Q = 1;
      while (Q < nseen + nnew) Q <<= 1;
      for (int i = nseen + nnew + threadIdx.x; i < Q; i += blockDim.x) cand[i] = INT_MAX;
      ap_bitonic(cand, Q);
      for (int i = threadIdx.x; i < nseen + nnew; i += blockDim.x) seen[i] = cand[i];
      __syncthreads();
      if (threadIdx.x == 0) {
        s_nseen = nseen + nnew;
        s_nfront = nnew;
      }
      __syncthreads();
    }
    if (s_bad) {
      if (threadIdx.x == 0) atomicExch(overflow, 1);
      __syncthreads();
      continue;
    }
    // pattern = seen U {col}, the lowest max_fill indices with col kept
    if (threadIdx.x == 0) {
      const int ns = s_nseen;
      const bool has = ap_contains(seen, ns, col);
      const int tot = ns + (has ? 0 : 1);
      const int keep = min(tot, max_fill);
      int* out = ipat + size_t(col) * max_fill;
      int o = 0, i = 0;
      bool placed = has;
      while (o < keep) {
        if (!placed && (i >= ns || col < seen[i])) {
          out[o++] = col;
          placed = true;
        } else {
          out[o++] = seen[i++];
        }
      }
      if (!ap_contains(out, keep, col)) {  // truncated past the diagonal: it replaces the largest kept index
        out[keep - 1] = col;
        for (int q = keep - 1; q > 0 && out[q] < out[q - 1]; --q) {
          const int t = out[q]; out[q] = out[q - 1]; out[q - 1] = t;
        }
      }
      icnt[col] = keep;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) k_spai(SpaiParams P) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  WarpWS w;
  {
    double* bd = P.wsd + size_t(gw) * P.ws_doubles;
    int* bi = P.wsi + size_t(gw) * P.ws_ints;
    w.D = bd; bd += size_t(P.IMAX) * P.PMAX;
    w.rhsl = bd; bd += P.IMAX;
    w.resid = bd; bd += P.IMAX + P.RHSMAX;
    w.coef = bd; bd += P.PMAX;
    w.hc = bd; bd += P.PMAX;
    w.upd = bd; bd += P.PMAX;
    w.dir = bd;
    w.J = bi; bi += P.PMAX;
    w.perm = bi; bi += P.PMAX;
    w.tr = bi; bi += P.PMAX;
    w.I = bi; bi += P.IMAX;
    w.I2 = bi; bi += P.IMAX;
    w.sb = bi;
  }
  while (true) {
    int col = 0;
    if (lane == 0) col = atomicAdd(P.next, 1);
    col = __shfl_sync(0xffffffffu, col, 0);
    if (P.only_col >= 0) {
      if (col > 0) return;
      col = P.only_col;
    }
    if (col >= P.n) return;
    // right-hand side
    const int* rr;
    const double* rv;
    int rn;
    int unit_row = col;
    double unit_val = 1.0;
    if (P.update) {
      const int b = P.prevt.rowptr[col], e = P.prevt.rowptr[col + 1];
      rr = P.prevt.colind + b;
      rv = P.prevt.val + b;
      rn = e - b;
      if (rn == 0) {  // zero target column: q = 0 exactly (chain.cpp:39-44)
        if (lane == 0) {
          P.cnt[col] = 1;
          P.orow[size_t(col) * P.PMAX] = col;
          P.oval[size_t(col) * P.PMAX] = 0.0;
          P.ores[col] = 0.0;
          P.ofb[col] = 0;
        }
        continue;
      }
    } else {
      rr = &unit_row;
      rv = &unit_val;
      rn = 1;
    }
    // initial pattern (spai.cpp:43-87): rows of A(:, col) U {col}, truncated
    int np = 0;
    {
      const int b = P.at.rowptr[col], e = P.at.rowptr[col + 1];
      if (P.fixed_J) {
        for (int i = lane; i < P.fixed_np; i += 32) w.J[i] = P.fixed_J[i];
        np = P.fixed_np;
      } else if (P.pattern_kind == 0) {
        if (lane == 0) w.J[0] = col;
        np = 1;
      } else if (P.pattern_kind == 2) {
        np = P.icnt[col];
        for (int i = lane; i < np; i += 32) w.J[i] = P.ipat[size_t(col) * P.istride + i];
      } else {
        // merge the sorted column rows with col
        const int len = e - b;
        const int pos = lower_bound_i(P.at.colind + b, len, col);
        const bool has = pos < len && P.at.colind[b + pos] == col;
        const int tot = len + (has ? 0 : 1);
        const int keep = min(tot, P.max_fill);
        for (int i = lane; i < keep; i += 32) {
          int v;
          if (has) v = P.at.colind[b + i];
          else v = i < pos ? P.at.colind[b + i] : (i == pos ? col : P.at.colind[b + i - 1]);
          w.J[i] = v;
        }
        __syncwarp();
        np = keep;
        if (tot > P.max_fill && lane == 0) {
          // keep the lowest indices plus the diagonal
          bool in = false;
          for (int i = 0; i < keep; ++i) in |= w.J[i] == col;
          if (!in) {
            w.J[keep - 1] = col;
            // re-sort (col is larger than all kept entries here)
            for (int i = keep - 1; i > 0 && w.J[i] < w.J[i - 1]; --i) {
              const int t = w.J[i]; w.J[i] = w.J[i - 1]; w.J[i - 1] = t;
            }
          }
        }
      }
      __syncwarp();
    }
    double rhs_norm2 = 0.0;
    for (int k = lane; k < rn; k += 32) rhs_norm2 = fma(rv[k], rv[k], rhs_norm2);
    rhs_norm2 = wsum(rhs_norm2);
    const double threshold = P.fill_tol * sqrt(rhs_norm2);
    // first solve
    // phase timing is a compile-time option (make EXTRA=-DMPG_SPAI_PHASES): the counters cost 24 registers
    // and spills (72 -> 96), 13 % of the C3 build time
#ifdef MPG_SPAI_PHASES
    long long tc0 = P.phase ? clock64() : 0, tc1, ph[4] = {0, 0, 0, 0};
#define MPG_PH(i)                 \
  if (P.phase) {                  \
    tc1 = clock64();              \
    ph[i] += tc1 - tc0;           \
    tc0 = tc1;                    \
  }
#else
#define MPG_PH(i)
#endif
    int m = build_rows(P, w, np, lane);
    MPG_PH(0)
    double outside_sq = 0.0;
    gather(P, w, np, m, rr, rv, rn, outside_sq, lane);
    MPG_PH(1)
    bool rankdef = qr_solve(w, m, np, lane);
    MPG_PH(2)
    double local_sq = residual_on_I(P, w, np, m, rr, rv, rn, lane);
    MPG_PH(3)
    double residual = sqrt(local_sq + outside_sq);
    for (int sweep = 0; sweep < P.max_sweeps; ++sweep) {
      if (residual <= threshold) break;
      if (np >= P.max_fill) break;
      // candidates: rows of I plus rhs rows outside I (outside residual = rhs value)
      double bv = 0.0;
      int bj = INT_MAX;
      for (int i = lane; i < m; i += 32) {
        const int row = w.I[i];
        const double mag = fabs(w.resid[i]);
        if (mag > bv || (mag == bv && mag > 0.0 && row < bj)) {
          const int jp = lower_bound_i(w.J, np, row);
          const bool in_pattern = jp < np && w.J[jp] == row;
          if (row < P.n && !in_pattern && P.at.rowptr[row + 1] > P.at.rowptr[row]) { bv = mag; bj = row; }
        }
      }
      for (int k = lane; k < rn; k += 32) {
        const int row = rr[k];
        const int pos = lower_bound_i(w.I, m, row);
        if (pos < m && w.I[pos] == row) continue;
        const double mag = fabs(rv[k]);
        if (mag > bv || (mag == bv && mag > 0.0 && row < bj)) {
          const int jp = lower_bound_i(w.J, np, row);
          if (row < P.n && (jp == np || w.J[jp] != row) && P.at.rowptr[row + 1] > P.at.rowptr[row]) {
            bv = mag;
            bj = row;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
      }
      if (!(bv > 0.0) || bj == INT_MAX) break;
      if (lane == 0) {
        int i = np;
        while (i > 0 && w.J[i - 1] > bj) { w.J[i] = w.J[i - 1]; --i; }
        w.J[i] = bj;
      }
      __syncwarp();
      ++np;
      MPG_PH(3)
      m = build_rows(P, w, np, lane);
      MPG_PH(0)
      gather(P, w, np, m, rr, rv, rn, outside_sq, lane);
      MPG_PH(1)
      rankdef = qr_solve(w, m, np, lane);
      MPG_PH(2)
      local_sq = residual_on_I(P, w, np, m, rr, rv, rn, lane);
      MPG_PH(3)
      residual = sqrt(local_sq + outside_sq);
    }
#undef MPG_PH
#ifdef MPG_SPAI_PHASES
    if (P.phase && lane == 0)
      for (int i = 0; i < 4; ++i) atomicAdd(P.phase + i, static_cast<unsigned long long>(ph[i]));
#endif
    if (rankdef && !P.raw) {
      if (!P.update) {
        // diagonal fallback (spai.cpp:196-218)
        const int b = P.at.rowptr[col], e = P.at.rowptr[col + 1];
        double diag = 0.0;
        int hit = 0;
        for (int k = b + lane; k < e; k += 32)
          if (P.at.colind[k] == col) { diag = P.at.val[k]; hit = 1; }
        diag = wsum(diag);
        hit = __reduce_or_sync(0xffffffffu, hit);
        const double coeff = diag != 0.0 ? 1.0 / diag : 1.0;
        double sq = 0.0;
        for (int k = b + lane; k < e; k += 32) {
          const double ev = (P.at.colind[k] == col ? 1.0 : 0.0) - coeff * P.at.val[k];
          sq = fma(ev, ev, sq);
        }
        sq = wsum(sq);
        if (!hit) sq += 1.0;
        if (lane == 0) {
          P.cnt[col] = 1;
          P.orow[size_t(col) * P.PMAX] = col;
          P.oval[size_t(col) * P.PMAX] = coeff;
          P.ores[col] = sqrt(sq);
          P.ofb[col] = 1;
        }
      } else {
        // identity fallback (chain.cpp:47-73): residual = ||prev(:,j) - new(:,j)||^2
        if (lane == 0) {
          const int b = P.at.rowptr[col], e = P.at.rowptr[col + 1];
          int pa = 0, pb = b;
          double sq = 0.0;
          while (pa < rn || pb < e) {
            if (pb >= e || (pa < rn && rr[pa] < P.at.colind[pb])) { sq += rv[pa] * rv[pa]; ++pa; }
            else if (pa >= rn || P.at.colind[pb] < rr[pa]) { sq += P.at.val[pb] * P.at.val[pb]; ++pb; }
            else { const double d = rv[pa] - P.at.val[pb]; sq += d * d; ++pa; ++pb; }
          }
          P.cnt[col] = 1;
          P.orow[size_t(col) * P.PMAX] = col;
          P.oval[size_t(col) * P.PMAX] = 1.0;
          P.ores[col] = sq;
          P.ofb[col] = 1;
        }
      }
    } else {
      for (int i = lane; i < np; i += 32) {
        P.orow[size_t(col) * P.PMAX + i] = w.J[i];
        P.oval[size_t(col) * P.PMAX + i] = w.coef[i];
      }
      if (lane == 0) {
        P.cnt[col] = np;
        P.ores[col] = P.update ? residual * residual : residual;
        P.ofb[col] = rankdef ? 1 : 0;
      }
    }
    __syncwarp();
  }
}

__global__ void k_compact(const int* __restrict__ cnt, const int* __restrict__ off, const int* __restrict__ orow,
                          const double* __restrict__ oval, int n, int PMAX, int* __restrict__ ci,
                          double* __restrict__ v) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int o = off[c];
  for (int i = 0; i < cnt[c]; ++i) {
    ci[o + i] = orow[size_t(c) * PMAX + i];
    v[o + i] = oval[size_t(c) * PMAX + i];
  }
}

__global__ void k_fro_dist(CsrView a, CsrView b, double* part) {
  __shared__ double red[8];
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.nrows; r += gridDim.x * blockDim.x) {
    int i = a.rowptr[r], j = b.rowptr[r];
    const int ie = a.rowptr[r + 1], je = b.rowptr[r + 1];
    while (i < ie || j < je) {
      double d;
      if (j >= je || (i < ie && a.colind[i] < b.colind[j])) d = a.val[i++];
      else if (i >= ie || b.colind[j] < a.colind[i]) d = -b.val[j++];
      else d = a.val[i++] - b.val[j++];
      s = fma(d, d, s);
    }
  }
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}

}  // namespace

double frobenius_distance(const CsrPtr& a, const CsrPtr& b) {
  auto& c = ctx(a->device);
  DeviceGuard g(a->device);
  const int blocks = 256;
  DBuf<double> part(a->device, blocks);
  k_fro_dist<<<blocks, 256, 0, c.stream>>>(a->view(), b->view(), part.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  std::vector<double> h(blocks);
  MPG_CUDA(cudaMemcpyAsync(h.data(), part.get(), blocks * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  double s = 0.0;
  for (double v : h) s += v;
  return std::sqrt(s);
}

SpaiOutcome spai_or_update(const CsrPtr& a, const CsrPtr& prev, const SpaiOptions& o, bool want_residuals) {
  const auto t0 = std::chrono::steady_clock::now();
  if (a->nrows != a->ncols) throw std::invalid_argument(prev ? "update_build: matrices must be square" : "spai_build: matrix must be square");
  if (prev && (prev->nrows != a->nrows || prev->ncols != a->ncols)) throw std::invalid_argument("update_build: shape mismatch");
  if (o.fill_tol < 0.0 || o.max_fill_per_col < 1 || o.max_pattern_sweeps < 0)
    throw std::invalid_argument("spai_build: invalid configuration");
  const int dev = a->device;
  auto& c = ctx(dev);
  DeviceGuard g(dev);
  cudaStream_t s = c.stream;
  const int n = int(a->nrows);
  SpaiOutcome out;
  if (n == 0) {
    DBuf<int> rp(dev, 1);
    MPG_CUDA(cudaMemsetAsync(rp.get(), 0, sizeof(int), s));
    out.p = csr_from_device_parts(dev, 0, 0, std::move(rp), DBuf<int>(), DBuf<double>());
    return out;
  }
  CsrPtr at = csr_transpose_cached(a);
  CsrPtr pt = prev ? csr_transpose_cached(prev) : nullptr;
  const int maxcol = at->max_row;
  const int maxrhs = pt ? pt->max_row : 1;
  // PatternOfAPow: the initial patterns are built first, on the device
  DBuf<int> ipat, icnt;
  int pinit = o.pattern_kind == 0 ? 1 : maxcol + 1;
  if (o.pattern_kind == 2) {
    ipat = DBuf<int>(dev, size_t(n) * size_t(o.max_fill_per_col));
    icnt = DBuf<int>(dev, size_t(n));
    DBuf<int> ovf(dev, 1);
    MPG_CUDA(cudaMemsetAsync(ovf.get(), 0, sizeof(int), s));
    k_apow_pattern<<<unsigned(std::min(n, c.sm_count * 8)), AP_THREADS, 0, s>>>(at->view(), o.power,
                                                                                o.max_fill_per_col, ipat.get(),
                                                                                icnt.get(), ovf.get());
    MPG_CHECK_LAUNCH();
    count_launch();
    int bad = 0;
    MPG_CUDA(cudaMemcpyAsync(&bad, ovf.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
    if (bad)
      throw ConfigError("spai: the A^" + std::to_string(o.power) + " pattern of a column exceeds " +
                        std::to_string(AP_SEEN) + " rows (or a frontier's supports " + std::to_string(AP_CAND) +
                        " entries) on the GPU path");
    pinit = o.max_fill_per_col;
  }
  const int PMAX = std::max(1, std::min(o.max_fill_per_col, pinit + o.max_pattern_sweeps));
  const int64_t imax64 = std::min<int64_t>(n, int64_t(PMAX) * std::max(maxcol, 1));
  const int IMAX = int(std::max<int64_t>(imax64, 1));
  int SORTN = 1;
  while (SORTN < PMAX * std::max(maxcol, 1)) SORTN <<= 1;
  const int RHSMAX = maxrhs;

  SpaiParams P{};
  P.at = at->view();
  P.prevt = pt ? pt->view() : CsrView{nullptr, nullptr, nullptr, 0, 0};
  P.n = n;
  P.update = prev ? 1 : 0;
  P.pattern_kind = o.pattern_kind;
  P.fill_tol = o.fill_tol;
  P.max_fill = o.max_fill_per_col;
  P.max_sweeps = o.max_pattern_sweeps;
  P.PMAX = PMAX;
  P.IMAX = IMAX;
  P.SORTN = SORTN;
  P.RHSMAX = RHSMAX;
  P.ws_doubles = (size_t(IMAX) * PMAX + 2 * size_t(IMAX) + RHSMAX + 4 * size_t(PMAX) + 1) & ~size_t(1);
  P.ws_ints = (3 * size_t(PMAX) + 2 * size_t(IMAX) + SORTN + 3) & ~size_t(3);
  // persistent grid, bounded by the workspace budget
  const size_t per_warp = P.ws_doubles * 8 + P.ws_ints * 4;
  // as many resident warps as the registers allow (the build is latency-bound:
  // C3 1.9 s at 16 warps/SM, 1.7 s at 28); MPG_SPAI_WPS overrides
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_spai, 128, 0) != cudaSuccess || bps < 1) {
    cudaGetLastError();
    bps = 4;
  }
  const int wps = std::getenv("MPG_SPAI_WPS") ? std::max(1, std::atoi(std::getenv("MPG_SPAI_WPS"))) : 4 * bps;
  int warps = c.sm_count * wps;
  const size_t budget = size_t(8) << 30;
  while (warps > c.sm_count && size_t(warps) * per_warp > budget) warps /= 2;
  warps = std::max(warps - warps % 4, 4);
  DBuf<double> wsd(dev, size_t(warps) * P.ws_doubles);
  DBuf<int> wsi(dev, size_t(warps) * P.ws_ints);
  DBuf<int> cnt(dev, size_t(n) + 1), orow(dev, size_t(n) * PMAX), ofb(dev, size_t(n)), next(dev, 1);
  DBuf<double> oval(dev, size_t(n) * PMAX), ores(dev, size_t(n));
  MPG_CUDA(cudaMemsetAsync(next.get(), 0, sizeof(int), s));
  P.wsd = wsd.get();
  P.wsi = wsi.get();
  P.cnt = cnt.get();
  P.orow = orow.get();
  P.oval = oval.get();
  P.ores = ores.get();
  P.ofb = ofb.get();
  P.next = next.get();
  P.fixed_J = nullptr;
  P.only_col = -1;
  P.raw = 0;
  P.ipat = ipat.get();
  P.icnt = icnt.get();
  P.istride = o.max_fill_per_col;
  DBuf<unsigned long long> phase;
#ifdef MPG_SPAI_PHASES
  if (std::getenv("MPG_SPAI_PHASES")) {
    phase = DBuf<unsigned long long>(dev, 4);
    MPG_CUDA(cudaMemsetAsync(phase.get(), 0, 4 * sizeof(unsigned long long), s));
    P.phase = phase.get();
  }
#endif
  k_spai<<<unsigned(warps / 4), 128, 0, s>>>(P);
  MPG_CHECK_LAUNCH();
  count_launch();
  if (P.phase) {
    unsigned long long h[4];
    MPG_CUDA(cudaMemcpyAsync(h, phase.get(), sizeof h, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
    const double tot = double(h[0] + h[1] + h[2] + h[3]) + 1.0;
    std::fprintf(stderr, "[mpg spai phases] warps %d  rows %.1f%%  gather %.1f%%  qr %.1f%%  residual+select %.1f%%\n", warps,
                 100.0 * h[0] / tot, 100.0 * h[1] / tot, 100.0 * h[2] / tot, 100.0 * h[3] / tot);
  }
  // CSR of P^T (column lists), then P = (P^T)^T on the device
  DBuf<int> off(dev, size_t(n) + 1);
  {
    MPG_CUDA(cudaMemsetAsync(cnt.get() + n, 0, sizeof(int), s));
    size_t tmp = 0;
    MPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), off.get(), n + 1, s));
    DBuf<char> t(dev, tmp);
    MPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, cnt.get(), off.get(), n + 1, s));
    count_launch();
  }
  int nnz = 0;
  MPG_CUDA(cudaMemcpyAsync(&nnz, off.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  DBuf<int> ci(dev, size_t(nnz));
  DBuf<double> vv(dev, size_t(nnz));
  k_compact<<<unsigned((n + 255) / 256), 256, 0, s>>>(cnt.get(), off.get(), orow.get(), oval.get(), n, PMAX, ci.get(),
                                                      vv.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  MPG_CUDA(cudaStreamSynchronize(s));
  CsrPtr ptr = csr_from_device_parts(dev, n, n, std::move(off), std::move(ci), std::move(vv));
  out.p = csr_transpose(*ptr);
  // residuals and fallbacks (summed on the host in column order, chain.cpp:86-93)
  std::vector<double> res(static_cast<size_t>(n));
  std::vector<int> fb(static_cast<size_t>(n));
  MPG_CUDA(cudaMemcpyAsync(res.data(), ores.get(), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaMemcpyAsync(fb.data(), ofb.get(), size_t(n) * sizeof(int), cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i) out.fallback_count += fb[size_t(i)];
  if (prev) {
    double tot = 0.0;
    for (double v : res) tot += v;
    out.min_residual = std::sqrt(tot);
    out.matrix_change = frobenius_distance(prev, a);
  }
  if (want_residuals) out.column_residuals = std::move(res);
  out.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}


void spai_column_solve_dev(const CsrPtr& a, int64_t col, const std::vector<int64_t>& pattern_in, std::vector<double>& values,
                           double& residual, bool& rank_def) {
  if (col < 0 || col >= a->ncols) throw std::invalid_argument("spai_column_solve: column out of range");
  std::vector<int> pat(pattern_in.begin(), pattern_in.end());
  std::sort(pat.begin(), pat.end());
  for (int v : pat)
    if (v < 0 || v >= a->ncols) throw std::invalid_argument("extract_column_submatrix: column index out of range");
  if (pat.empty()) throw std::invalid_argument("extract_column_submatrix: empty pattern");
  if (std::adjacent_find(pat.begin(), pat.end()) != pat.end())
    throw std::invalid_argument("extract_column_submatrix: repeated pattern index");
  const int dev = a->device;
  auto& c = ctx(dev);
  DeviceGuard g(dev);
  cudaStream_t s = c.stream;
  const int n = int(a->nrows);
  CsrPtr at = csr_transpose_cached(a);
  const int np = int(pat.size());
  const int maxcol = std::max(at->max_row, 1);
  SpaiParams P{};
  P.at = at->view();
  P.prevt = CsrView{nullptr, nullptr, nullptr, 0, 0};
  P.n = n;
  P.pattern_kind = 1;
  P.max_fill = np;
  P.max_sweeps = 0;
  P.PMAX = np;
  P.IMAX = int(std::min<int64_t>(n, int64_t(np) * maxcol));
  int SORTN = 1;
  while (SORTN < np * maxcol) SORTN <<= 1;
  P.SORTN = SORTN;
  P.RHSMAX = 1;
  P.ws_doubles = (size_t(P.IMAX) * np + 2 * size_t(P.IMAX) + 1 + 4 * size_t(np) + 1) & ~size_t(1);
  P.ws_ints = (3 * size_t(np) + 2 * size_t(P.IMAX) + SORTN + 3) & ~size_t(3);
  DBuf<double> wsd(dev, 4 * P.ws_doubles), oval(dev, size_t(n) * np), ores(dev, size_t(n));
  DBuf<int> wsi(dev, 4 * P.ws_ints), cnt(dev, size_t(n)), orow(dev, size_t(n) * np), ofb(dev, size_t(n)), next(dev, 1),
      fj(dev, size_t(np));
  MPG_CUDA(cudaMemsetAsync(next.get(), 0, sizeof(int), s));
  MPG_CUDA(cudaMemcpyAsync(fj.get(), pat.data(), pat.size() * 4, cudaMemcpyHostToDevice, s));
  P.wsd = wsd.get(); P.wsi = wsi.get(); P.cnt = cnt.get(); P.orow = orow.get(); P.oval = oval.get();
  P.ores = ores.get(); P.ofb = ofb.get(); P.next = next.get();
  P.fixed_J = fj.get(); P.fixed_np = np; P.only_col = int(col); P.raw = 1;
  k_spai<<<1, 128, 0, s>>>(P);
  MPG_CHECK_LAUNCH();
  count_launch();
  values.resize(size_t(np));
  int fb = 0;
  MPG_CUDA(cudaMemcpyAsync(values.data(), oval.get() + size_t(col) * np, size_t(np) * 8, cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaMemcpyAsync(&residual, ores.get() + col, 8, cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaMemcpyAsync(&fb, ofb.get() + col, 4, cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  rank_def = fb != 0;
}

}  // namespace mpg
