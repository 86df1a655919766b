// K1 / K1T / K1c: fused shifted SpMV y = s (sigma E - A) x formed on the fly
// (replaces linear_combination at proj/src/qbihomm.cpp:164-171 and the N = 0
// KroneckerOperator::apply, proj/src/kron.cpp:34-64), plain CSR SpMV
// (SparseMatrix::multiply, proj/src/sparse.cpp:236-249), the device transpose
// (the CSC shadow, sparse.cpp:27-46 / 289-299), chain application
// (PrecondChain::apply, proj/src/chain.cpp:117-126) and the explicit unit
// operator (assemble_explicit, proj/src/kron.cpp:72-131).
//
// Roofline: HBM-bound. Per shifted SpMV: 12 nnz(A) + 4(n+1) + B_E + 16 n bytes
// (B_E = 8n diagonal, 8 nnz(A) for E sharing A's pattern) — DESIGN.md §6.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>

#include "runtime.cuh"

namespace mpg {

std::atomic<long long> g_launches{0};

namespace {
std::atomic<bool> g_prof_on{false};
std::mutex g_prof_mu;
struct ProfEntry { long long launches = 0; double ms = 0.0, bytes = 0.0; };
ProfEntry g_prof[PK_COUNT];
}  // namespace

bool profile_enabled() { return g_prof_on.load(); }
void profile_set(bool on) { g_prof_on.store(on); }
void profile_reset() {
  std::scoped_lock l(g_prof_mu);
  for (auto& e : g_prof) e = ProfEntry{};
}
void profile_add(int kind, double ms, long long launches) {
  std::scoped_lock l(g_prof_mu);
  g_prof[kind].ms += ms;
  g_prof[kind].launches += launches;
}
void profile_add_bytes(int kind, double bytes) {
  std::scoped_lock l(g_prof_mu);
  g_prof[kind].bytes += bytes;
}
void profile_read(int kind, long long* launches, double* ms, double* bytes) {
  std::scoped_lock l(g_prof_mu);
  *launches = g_prof[kind].launches;
  *ms = g_prof[kind].ms;
  *bytes = g_prof[kind].bytes;
}

DeviceCtx& ctx(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<DeviceCtx>> ctxs;
  std::scoped_lock l(mu);
  auto& slot = ctxs[device];
  if (!slot) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw CudaError("no CUDA device available");
    if (device < 0 || device >= count) throw CudaError("device index out of range");
    DeviceGuard g(device);
    auto c = std::make_unique<DeviceCtx>();
    c->device = device;
    MPG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    MPG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    cudaMemPool_t pool;
    MPG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    MPG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    slot = std::move(c);
  }
  return *slot;
}

void* dmalloc(int device, size_t bytes) {
  DeviceGuard g(device);
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, ctx(device).stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    MPG_CUDA(cudaStreamSynchronize(ctx(device).stream));
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, device);
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&p, bytes, ctx(device).stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
  }
  return p;
}

void dfree(int device, void* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaFreeAsync(p, ctx(device).stream);
  cudaSetDevice(prev);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void copy_in(double* dst, const double* src, size_t n, cudaStream_t s) {
  if (n) MPG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, s));
}
void copy_out(double* dst, const double* src, size_t n, cudaStream_t s) {
  if (n) MPG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, s));
}

int choose_vec_width(double mean_row) {
  static const int forced = [] {
    const char* e = std::getenv("MPG_VEC_WIDTH");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
  // About four entries per lane: enough independent loads in flight per lane
  // and log2(V) shuffle steps per row.
  // (measured on the 27-point C3 operator: V = 4 beats 8/16/32 by 1.4-3x).
  if (mean_row > 128) return 32;
  if (mean_row > 64) return 16;
  if (mean_row > 32) return 8;
  if (mean_row > 5) return 4;
  return 2;
}

// ---------------------------------------------------------------------------
// kernels
namespace {

template <int V>
__device__ __forceinline__ double sub_sum(double v) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, V);
  return v;
}

// V = 0: the row-binned mapping (runtime.cuh bin_locate), sub-warp width per block.
template <int V>
__global__ void __launch_bounds__(256) k_spmv(CsrView m, const double* __restrict__ x, double* __restrict__ y,
                                              double alpha) {
  int lane, row, W = V;
  bool ok;
  if (V == 0) {
    ok = bin_locate(m, row, W, lane);
  } else {
    lane = threadIdx.x & (V - 1);
    row = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) / V);
    ok = row < m.nrows;
  }
  double acc = 0.0;
  if (ok) {
    const int b = m.rowptr[row], e = m.rowptr[row + 1];
#pragma unroll 4
    for (int k = b + lane; k < e; k += W) acc = fma(__ldcs(m.val + k), __ldg(x + __ldcs(m.colind + k)), acc);
  }
  acc = V ? sub_sum<(V ? V : 2)>(acc) : sub_sum_rt(acc, W);
  if (ok && lane == 0) y[row] = alpha * acc;
}

// y = s (sigma E x + ca A x); PAIR: 2n real form; RESID: y = resid - (...)
template <int V, int EM, bool PAIR>
__global__ void __launch_bounds__(256) k_op(OpView op, double sre, double sim, double ca, const double* __restrict__ x,
                                            double* __restrict__ y, const double* __restrict__ resid, double scale) {
  const int n = op.a.nrows;
  int lane, row, W = V;
  bool ok;
  if (V == 0) {  // row-binned mapping
    ok = bin_locate(op.a, row, W, lane);
  } else {
    lane = threadIdx.x & (V - 1);
    row = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) / V);
    ok = row < n;
  }
  double a1 = 0.0, a2 = 0.0, e1 = 0.0, e2 = 0.0;
  if (ok) {
    const int b = op.a.rowptr[row], e = op.a.rowptr[row + 1];
    if (EM == E_SAMEPAT) {
#pragma unroll 4
      for (int k = b + lane; k < e; k += W) {
        const double2 ae = __ldcs(op.ae + k);
        const int c = __ldcs(op.a.colind + k);
        const double x1 = __ldg(x + c);
        a1 = fma(ae.x, x1, a1);
        e1 = fma(ae.y, x1, e1);
        if (PAIR) {
          const double x2 = __ldg(x + n + c);
          a2 = fma(ae.x, x2, a2);
          e2 = fma(ae.y, x2, e2);
        }
      }
    } else {
#pragma unroll 4
      for (int k = b + lane; k < e; k += W) {
        const double av = __ldcs(op.a.val + k);
        const int c = __ldcs(op.a.colind + k);
        a1 = fma(av, __ldg(x + c), a1);
        if (PAIR) a2 = fma(av, __ldg(x + n + c), a2);
      }
    }
  }
#define MPG_SUBSUM(v) v = V ? sub_sum<(V ? V : 2)>(v) : sub_sum_rt(v, W)
  MPG_SUBSUM(a1);
  if (PAIR) MPG_SUBSUM(a2);
  if (EM == E_SAMEPAT) {
    MPG_SUBSUM(e1);
    if (PAIR) MPG_SUBSUM(e2);
  }
#undef MPG_SUBSUM
  if (ok && lane == 0) {
    if (EM == E_IDENT) {
      e1 = x[row];
      if (PAIR) e2 = x[n + row];
    } else if (EM == E_DIAG) {
      const double d = op.ediag[row];
      e1 = d * x[row];
      if (PAIR) e2 = d * x[n + row];
    }
    if (PAIR) {
      const double y1 = sre * e1 + ca * a1 + sim * e2;
      const double y2 = -sim * e1 + sre * e2 + ca * a2;
      if (resid) {
        y[row] = resid[row] - y1;
        y[n + row] = resid[n + row] - y2;
      } else {
        y[row] = scale * y1;
        y[n + row] = scale * y2;
      }
    } else {
      const double y1 = sre * e1 + ca * a1;
      y[row] = resid ? resid[row] - y1 : scale * y1;
    }
  }
}

__global__ void k_row_index(const int* __restrict__ rp, int nrows, int* __restrict__ rows) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  for (int k = rp[r]; k < rp[r + 1]; ++k) rows[k] = r;
}

__global__ void k_iota(int* p, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = int(i);
}

__global__ void k_count(const int* __restrict__ keys, int64_t nnz, int* __restrict__ counts) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < nnz) atomicAdd(counts + keys[i], 1);
}

__global__ void k_gather_t(const int* __restrict__ perm, const int* __restrict__ rows, const double* __restrict__ val,
                           int64_t nnz, int* __restrict__ tci, double* __restrict__ tval) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nnz) return;
  const int k = perm[i];
  tci[i] = rows[k];
  tval[i] = val[k];
}

__global__ void k_stats(const int* __restrict__ rp, const int* __restrict__ ci, int nrows, int* __restrict__ out) {
  // out[0] = max row length, out[1] = number of rows that are not exactly {i}
  int mx = 0, notdiag = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int len = rp[r + 1] - rp[r];
    mx = max(mx, len);
    if (!(len == 1 && ci[rp[r]] == r)) ++notdiag;
  }
  atomicMax(out, mx);
  if (notdiag) atomicAdd(out + 1, notdiag);
}

// Row bins: class key and identity index per row, class histogram.
__global__ void k_bin_key(const int* __restrict__ rp, int nrows, unsigned char* __restrict__ key,
                          int* __restrict__ idx, int* __restrict__ hist) {
  __shared__ int sh[NBIN];
  if (threadIdx.x < NBIN) sh[threadIdx.x] = 0;
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrows) {
    const int b = row_bin(rp[r + 1] - rp[r]);
    key[r] = static_cast<unsigned char>(b);
    idx[r] = r;
    atomicAdd(sh + b, 1);
  }
  __syncthreads();
  if (threadIdx.x < NBIN && sh[threadIdx.x]) atomicAdd(hist + threadIdx.x, sh[threadIdx.x]);
}

__global__ void k_sq_partial(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s = fma(x[i], x[i], s);
  s = sub_sum<32>(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
    s = sub_sum<32>(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void k_sum_partial(const double* __restrict__ part, int n, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) s += part[i];
  s = sub_sum<32>(s);
  if (threadIdx.x == 0) *out = s;
}

// Explicit unit operator: counts per output row.
__global__ void k_expl_count(CsrView a, CsrView e, int emode, int pair, int* __restrict__ counts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  // merged pattern of A(r, :) and E(r, :) (E_IDENT / E_DIAG: the diagonal)
  int na = a.rowptr[r + 1] - a.rowptr[r];
  int cnt = 0, ne = 0;
  if (emode == E_IDENT || emode == E_DIAG) {
    bool has = false;
    for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) has |= a.colind[k] == r;
    cnt = na + (has ? 0 : 1);
    ne = 1;
  } else {  // E_SAMEPAT: identical pattern
    cnt = na;
    ne = na;
  }
  if (!pair) {
    counts[r] = cnt;
  } else {
    counts[r] = cnt + ne;
    counts[a.nrows + r] = ne + cnt;
  }
}

__device__ __forceinline__ void emit_merged(CsrView a, const double2* ae, const double* ediag, int emode, int r,
                                            double sre, double ca, int coloff, int* __restrict__ ci,
                                            double* __restrict__ v, int& p) {
  if (emode == E_SAMEPAT) {
    for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
      ci[p] = a.colind[k] + coloff;
      v[p] = sre * ae[k].y + ca * ae[k].x;
      ++p;
    }
    return;
  }
  const double d = emode == E_DIAG ? ediag[r] : 1.0;
  bool done = false;
  for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
    const int c = a.colind[k];
    if (!done && c > r) {
      ci[p] = r + coloff;
      v[p] = sre * d;
      ++p;
      done = true;
    }
    if (c == r) {
      ci[p] = c + coloff;
      v[p] = sre * d + ca * a.val[k];
      ++p;
      done = true;
    } else {
      ci[p] = c + coloff;
      v[p] = ca * a.val[k];
      ++p;
    }
  }
  if (!done) {
    ci[p] = r + coloff;
    v[p] = sre * d;
    ++p;
  }
}

__device__ __forceinline__ void emit_e(CsrView a, const double2* ae, const double* ediag, int emode, int r, double s,
                                       int coloff, int* __restrict__ ci, double* __restrict__ v, int& p) {
  if (emode == E_SAMEPAT) {
    for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
      ci[p] = a.colind[k] + coloff;
      v[p] = s * ae[k].y;
      ++p;
    }
  } else {
    ci[p] = r + coloff;
    v[p] = s * (emode == E_DIAG ? ediag[r] : 1.0);
    ++p;
  }
}

__global__ void k_expl_fill(CsrView a, const double2* ae, const double* ediag, int emode, int pair, double sre,
                            double sim, const int* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = a.nrows;
  if (r >= n) return;
  int p = rp[r];
  emit_merged(a, ae, ediag, emode, r, sre, -1.0, 0, ci, v, p);
  if (pair) {
    emit_e(a, ae, ediag, emode, r, sim, n, ci, v, p);
    int q = rp[n + r];
    emit_e(a, ae, ediag, emode, r, -sim, 0, ci, v, q);
    emit_merged(a, ae, ediag, emode, r, sre, -1.0, n, ci, v, q);
  }
}

__global__ void k_interleave(const double* __restrict__ a, const double* __restrict__ e, int64_t nnz,
                             double2* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < nnz) out[i] = make_double2(a[i], e[i]);
}

// Merge A and E (general patterns) into the union pattern, values interleaved.
__global__ void k_union_count(CsrView a, CsrView e, int* __restrict__ counts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  int i = a.rowptr[r], j = e.rowptr[r], ie = a.rowptr[r + 1], je = e.rowptr[r + 1], c = 0;
  while (i < ie || j < je) {
    if (j >= je || (i < ie && a.colind[i] < e.colind[j])) ++i;
    else if (i >= ie || e.colind[j] < a.colind[i]) ++j;
    else { ++i; ++j; }
    ++c;
  }
  counts[r] = c;
}

__global__ void k_union_fill(CsrView a, CsrView e, const int* __restrict__ rp, int* __restrict__ ci,
                             double* __restrict__ av, double2* __restrict__ aev) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  int i = a.rowptr[r], j = e.rowptr[r], ie = a.rowptr[r + 1], je = e.rowptr[r + 1], p = rp[r];
  while (i < ie || j < je) {
    double x = 0.0, y = 0.0;
    int c;
    if (j >= je || (i < ie && a.colind[i] < e.colind[j])) { c = a.colind[i]; x = a.val[i++]; }
    else if (i >= ie || e.colind[j] < a.colind[i]) { c = e.colind[j]; y = e.val[j++]; }
    else { c = a.colind[i]; x = a.val[i++]; y = e.val[j++]; }
    ci[p] = c;
    av[p] = x;
    aev[p] = make_double2(x, y);
    ++p;
  }
}

inline unsigned grid_for(int64_t threads, int block = 256) { return unsigned((threads + block - 1) / block); }

void exclusive_scan(int device, const int* counts, int* out, int n, cudaStream_t s) {
  size_t tmp = 0;
  MPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, out, n + 1, s));
  DBuf<char> t(device, tmp);
  MPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, counts, out, n + 1, s));
  count_launch();
}

}  // namespace

// ---------------------------------------------------------------------------
void csr_finalize_stats(DevCsr& m) {
  auto& c = ctx(m.device);
  DeviceGuard g(m.device);
  m.mean_row = m.nrows ? double(m.nnz) / double(m.nrows) : 0.0;
  if (m.nrows == 0) return;
  DBuf<int> st(m.device, 2);
  MPG_CUDA(cudaMemsetAsync(st.get(), 0, 2 * sizeof(int), c.stream));
  k_stats<<<std::min<unsigned>(grid_for(m.nrows), 1184), 256, 0, c.stream>>>(m.rowptr.get(), m.colind.get(),
                                                                               int(m.nrows), st.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  int h[2];
  MPG_CUDA(cudaMemcpyAsync(h, st.get(), sizeof h, cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  m.max_row = h[0];
  m.is_diag = m.nrows == m.ncols && h[1] == 0;
  // Row bins for irregular matrices (the long-row split; runtime.cuh): the
  // longest row far above the mean means a fixed sub-warp width leaves most
  // lanes of a warp idle while one of its rows runs on.
  static const int bins_env = [] {
    const char* e = std::getenv("MPG_ROW_BINS");
    return e ? std::atoi(e) : -1;  // 0: never, 1: always, default: by the row statistics
  }();
  const bool want = bins_env == 1 || (bins_env != 0 && m.max_row > 64 && double(m.max_row) > 4.0 * m.mean_row);
  if (!want) return;
  const int n = int(m.nrows);
  DBuf<unsigned char> key(m.device, size_t(n)), key2(m.device, size_t(n));
  DBuf<int> idx(m.device, size_t(n)), hist(m.device, NBIN);
  m.brow = DBuf<int>(m.device, size_t(n));
  MPG_CUDA(cudaMemsetAsync(hist.get(), 0, NBIN * sizeof(int), c.stream));
  k_bin_key<<<grid_for(n), 256, 0, c.stream>>>(m.rowptr.get(), n, key.get(), idx.get(), hist.get());
  MPG_CHECK_LAUNCH();
  size_t tmp = 0;
  MPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), key2.get(), idx.get(), m.brow.get(), n, 0, 3,
                                           c.stream));
  DBuf<char> t(m.device, tmp);
  MPG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), key2.get(), idx.get(), m.brow.get(), n, 0, 3,
                                           c.stream));
  count_launch(2);
  int hh[NBIN];
  MPG_CUDA(cudaMemcpyAsync(hh, hist.get(), sizeof hh, cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  m.boff[0] = m.bblk[0] = 0;
  for (int b = 0; b < NBIN; ++b) {
    m.boff[b + 1] = m.boff[b] + hh[b];
    m.bblk[b + 1] = m.bblk[b] + int((int64_t(hh[b]) * (2 << b) + 255) / 256);
  }
}

CsrPtr csr_from_host(int device, int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci, const double* v) {
  // Validation as SparseMatrix::from_csr (proj/src/sparse.cpp:48-74).
  if (nr < 0 || nc < 0) throw std::invalid_argument("sparse: negative dimension");
  if (!rp) throw std::invalid_argument("sparse: row_offsets must not be null");
  if (rp[0] != 0) throw std::invalid_argument("sparse: row_offsets must start at 0");
  const int64_t nnz = rp[nr];
  if (nnz >= (int64_t(1) << 31) || nr >= (int64_t(1) << 31) - 1 || nc >= (int64_t(1) << 31) - 1)
    throw std::invalid_argument("sparse: int32 index range exceeded");
  for (int64_t i = 0; i < nr; ++i) {
    const int64_t lo = rp[i], hi = rp[i + 1];
    if (hi < lo) throw std::invalid_argument("sparse: row_offsets must be nondecreasing");
    int64_t prev = -1;
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t j = ci[k];
      if (j < 0 || j >= nc) throw std::invalid_argument("sparse: column index out of range in row " + std::to_string(i));
      if (j <= prev)
        throw std::invalid_argument("sparse: column indices must be strictly increasing in row " + std::to_string(i));
      prev = j;
    }
  }
  auto& c = ctx(device);
  DeviceGuard g(device);
  std::vector<int> rp32(size_t(nr) + 1), ci32(static_cast<size_t>(nnz));
  for (int64_t i = 0; i <= nr; ++i) rp32[size_t(i)] = int(rp[i]);
  for (int64_t k = 0; k < nnz; ++k) ci32[size_t(k)] = int(ci[k]);
  DBuf<int> drp(device, size_t(nr) + 1), dci(device, size_t(nnz));
  DBuf<double> dv(device, size_t(nnz));
  MPG_CUDA(cudaMemcpyAsync(drp.get(), rp32.data(), rp32.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  if (nnz) {
    MPG_CUDA(cudaMemcpyAsync(dci.get(), ci32.data(), ci32.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    MPG_CUDA(cudaMemcpyAsync(dv.get(), v, size_t(nnz) * sizeof(double), cudaMemcpyDefault, c.stream));
  }
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return csr_from_device_parts(device, nr, nc, std::move(drp), std::move(dci), std::move(dv));
}

CsrPtr csr_from_device_parts(int device, int64_t nr, int64_t nc, DBuf<int>&& rp, DBuf<int>&& ci, DBuf<double>&& v) {
  auto m = std::make_shared<DevCsr>();
  m->device = device;
  m->nrows = nr;
  m->ncols = nc;
  m->nnz = int64_t(ci.n);
  m->rowptr = std::move(rp);
  m->colind = std::move(ci);
  m->val = std::move(v);
  csr_finalize_stats(*m);
  return m;
}

CsrPtr csr_transpose(const DevCsr& a) {
  auto& c = ctx(a.device);
  DeviceGuard g(a.device);
  const int64_t nnz = a.nnz;
  DBuf<int> trp(a.device, size_t(a.ncols) + 1), tci(a.device, size_t(nnz));
  DBuf<double> tv(a.device, size_t(nnz));
  DBuf<int> counts(a.device, size_t(a.ncols) + 1);
  MPG_CUDA(cudaMemsetAsync(counts.get(), 0, (size_t(a.ncols) + 1) * sizeof(int), c.stream));
  if (nnz) {
    k_count<<<grid_for(nnz), 256, 0, c.stream>>>(a.colind.get(), nnz, counts.get());
    MPG_CHECK_LAUNCH();
    count_launch();
  }
  exclusive_scan(a.device, counts.get(), trp.get(), int(a.ncols), c.stream);
  if (nnz) {
    // Stable radix sort of (column, position) keeps rows ascending inside each
    // transposed row, exactly like the row-major shadow fill (sparse.cpp:38-45).
    DBuf<int> rows(a.device, size_t(nnz)), idx(a.device, size_t(nnz)), keys2(a.device, size_t(nnz)),
        idx2(a.device, size_t(nnz));
    k_row_index<<<grid_for(a.nrows), 256, 0, c.stream>>>(a.rowptr.get(), int(a.nrows), rows.get());
    MPG_CHECK_LAUNCH();
    k_iota<<<grid_for(nnz), 256, 0, c.stream>>>(idx.get(), nnz);
    MPG_CHECK_LAUNCH();
    count_launch(2);
    int bits = 1;
    while ((int64_t(1) << bits) < a.ncols) ++bits;
    size_t tmp = 0;
    MPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a.colind.get(), keys2.get(), idx.get(), idx2.get(),
                                             int64_t(nnz), 0, bits, c.stream));
    DBuf<char> t(a.device, tmp);
    MPG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, a.colind.get(), keys2.get(), idx.get(), idx2.get(),
                                             int64_t(nnz), 0, bits, c.stream));
    count_launch();
    k_gather_t<<<grid_for(nnz), 256, 0, c.stream>>>(idx2.get(), rows.get(), a.val.get(), nnz, tci.get(), tv.get());
    MPG_CHECK_LAUNCH();
    count_launch();
    MPG_CUDA(cudaStreamSynchronize(c.stream));
  }
  return csr_from_device_parts(a.device, a.ncols, a.nrows, std::move(trp), std::move(tci), std::move(tv));
}

CsrPtr csr_transpose_cached(const CsrPtr& a) {
  std::scoped_lock l(a->mu);
  if (!a->tcache) a->tcache = csr_transpose(*a);
  return a->tcache;
}

OpView ShiftedOp::view(bool transpose) const {
  OpView v{};
  const CsrPtr& m = transpose ? at : a;
  v.a = m->view();
  v.emode = emode;
  v.ediag = ediag.get();
  v.ae = transpose ? ae_t.get() : ae.get();
  return v;
}

OpPtr op_create(const CsrPtr& a, const CsrPtr& e) {
  if (a->nrows != a->ncols) throw std::invalid_argument("operator: A must be square");
  if (e && (e->nrows != a->nrows || e->ncols != a->ncols)) throw std::invalid_argument("operator: E must match A");
  if (e && e->device != a->device) throw std::invalid_argument("operator: A and E on different devices");
  auto& c = ctx(a->device);
  DeviceGuard g(a->device);
  auto op = std::make_shared<ShiftedOp>();
  op->device = a->device;
  op->n = a->nrows;
  op->a = a;
  op->e = e;
  if (!e) {
    op->emode = E_IDENT;
    op->at = csr_transpose_cached(a);
  } else if (e->is_diag) {
    op->emode = E_DIAG;
    op->ediag = DBuf<double>(a->device, size_t(a->nrows));
    MPG_CUDA(cudaMemcpyAsync(op->ediag.get(), e->val.get(), size_t(a->nrows) * sizeof(double),
                             cudaMemcpyDeviceToDevice, c.stream));
    op->at = csr_transpose_cached(a);
  } else {
    // E sharing A's pattern is interleaved directly; a general E is merged with
    // A into the union pattern (zero-filled) and then treated the same way.
    bool same = e->nnz == a->nnz;
    if (same) {
      std::vector<int> r1(size_t(a->nrows) + 1), r2(size_t(a->nrows) + 1), c1(size_t(a->nnz)), c2(size_t(a->nnz));
      MPG_CUDA(cudaMemcpyAsync(r1.data(), a->rowptr.get(), r1.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaMemcpyAsync(r2.data(), e->rowptr.get(), r2.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaMemcpyAsync(c1.data(), a->colind.get(), c1.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaMemcpyAsync(c2.data(), e->colind.get(), c2.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaStreamSynchronize(c.stream));
      same = r1 == r2 && c1 == c2;
    }
    CsrPtr au = a, eu = e;
    if (!same) {
      const int n = int(a->nrows);
      DBuf<int> counts(a->device, size_t(n) + 1), rp(a->device, size_t(n) + 1);
      MPG_CUDA(cudaMemsetAsync(counts.get(), 0, (size_t(n) + 1) * sizeof(int), c.stream));
      k_union_count<<<grid_for(n), 256, 0, c.stream>>>(a->view(), e->view(), counts.get());
      MPG_CHECK_LAUNCH();
      count_launch();
      exclusive_scan(a->device, counts.get(), rp.get(), n, c.stream);
      int nnz = 0;
      MPG_CUDA(cudaMemcpyAsync(&nnz, rp.get() + n, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaStreamSynchronize(c.stream));
      DBuf<int> ci(a->device, size_t(nnz));
      DBuf<double> av(a->device, size_t(nnz)), ev(a->device, size_t(nnz));
      DBuf<double2> aev(a->device, size_t(nnz));
      k_union_fill<<<grid_for(n), 256, 0, c.stream>>>(a->view(), e->view(), rp.get(), ci.get(), av.get(), aev.get());
      MPG_CHECK_LAUNCH();
      count_launch();
      DBuf<int> rp2(a->device, size_t(n) + 1), ci2(a->device, size_t(nnz));
      MPG_CUDA(cudaMemcpyAsync(rp2.get(), rp.get(), (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, c.stream));
      MPG_CUDA(cudaMemcpyAsync(ci2.get(), ci.get(), size_t(nnz) * 4, cudaMemcpyDeviceToDevice, c.stream));
      // E values along the union pattern
      std::vector<double2> h(static_cast<size_t>(nnz));
      MPG_CUDA(cudaMemcpyAsync(h.data(), aev.get(), size_t(nnz) * sizeof(double2), cudaMemcpyDeviceToHost, c.stream));
      MPG_CUDA(cudaStreamSynchronize(c.stream));
      std::vector<double> eh(static_cast<size_t>(nnz));
      for (int k = 0; k < nnz; ++k) eh[size_t(k)] = h[size_t(k)].y;
      MPG_CUDA(cudaMemcpyAsync(ev.get(), eh.data(), size_t(nnz) * 8, cudaMemcpyHostToDevice, c.stream));
      au = csr_from_device_parts(a->device, n, n, std::move(rp), std::move(ci), std::move(av));
      eu = csr_from_device_parts(a->device, n, n, std::move(rp2), std::move(ci2), std::move(ev));
      op->a = au;
    }
    op->emode = E_SAMEPAT;
    op->ae = DBuf<double2>(a->device, size_t(au->nnz));
    if (au->nnz) {
      k_interleave<<<grid_for(au->nnz), 256, 0, c.stream>>>(au->val.get(), eu->val.get(), au->nnz, op->ae.get());
      MPG_CHECK_LAUNCH();
      count_launch();
    }
    op->at = csr_transpose_cached(au);
    op->et = csr_transpose_cached(eu);
    op->ae_t = DBuf<double2>(a->device, size_t(au->nnz));
    if (au->nnz) {
      k_interleave<<<grid_for(au->nnz), 256, 0, c.stream>>>(op->at->val.get(), op->et->val.get(), au->nnz,
                                                             op->ae_t.get());
      MPG_CHECK_LAUNCH();
      count_launch();
    }
  }
  op->vec_width = choose_vec_width(op->a->mean_row);
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return op;
}

template <int V>
static void launch_spmv_v(const DevCsr& m, const double* x, double* y, double alpha, cudaStream_t s) {
  k_spmv<V><<<grid_for(m.nrows * int64_t(V)), 256, 0, s>>>(m.view(), x, y, alpha);
  MPG_CHECK_LAUNCH();
  count_launch();
}

void launch_spmv(const DevCsr& m, const double* x, double* y, double alpha, cudaStream_t s) {
  if (m.nrows == 0) return;
  if (m.brow.get()) {
    k_spmv<0><<<unsigned(m.bblk[NBIN]), 256, 0, s>>>(m.view(), x, y, alpha);
    MPG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  switch (choose_vec_width(m.mean_row)) {
    case 2: launch_spmv_v<2>(m, x, y, alpha, s); break;
    case 4: launch_spmv_v<4>(m, x, y, alpha, s); break;
    case 8: launch_spmv_v<8>(m, x, y, alpha, s); break;
    case 16: launch_spmv_v<16>(m, x, y, alpha, s); break;
    default: launch_spmv_v<32>(m, x, y, alpha, s); break;
  }
}

template <int V, int EM>
static void launch_op_ve(const OpView& v, int64_t n, double sre, double sim, double ca, const double* x, double* y,
                         const double* resid, double scale, cudaStream_t s) {
  const unsigned grid = V ? grid_for(n * int64_t(V)) : unsigned(v.a.bblk[NBIN]);
  if (sim != 0.0) k_op<V, EM, true><<<grid, 256, 0, s>>>(v, sre, sim, ca, x, y, resid, scale);
  else k_op<V, EM, false><<<grid, 256, 0, s>>>(v, sre, sim, ca, x, y, resid, scale);
  MPG_CHECK_LAUNCH();
  count_launch();
}

template <int V>
static void launch_op_v(const OpView& v, int64_t n, double sre, double sim, double ca, const double* x, double* y,
                        const double* resid, double scale, cudaStream_t s) {
  switch (v.emode) {
    case E_IDENT: launch_op_ve<V, E_IDENT>(v, n, sre, sim, ca, x, y, resid, scale, s); break;
    case E_DIAG: launch_op_ve<V, E_DIAG>(v, n, sre, sim, ca, x, y, resid, scale, s); break;
    default: launch_op_ve<V, E_SAMEPAT>(v, n, sre, sim, ca, x, y, resid, scale, s); break;
  }
}

void launch_op(const ShiftedOp& op, bool transpose, double sre, double sim, double ca, const double* x, double* y,
               const double* resid, double scale, cudaStream_t s, double* /*tmp_general*/) {
  if (op.n == 0) return;
  const OpView v = op.view(transpose);
  if (v.a.brow) {
    launch_op_v<0>(v, op.n, sre, sim, ca, x, y, resid, scale, s);
    return;
  }
  switch (op.vec_width) {
    case 2: launch_op_v<2>(v, op.n, sre, sim, ca, x, y, resid, scale, s); break;
    case 4: launch_op_v<4>(v, op.n, sre, sim, ca, x, y, resid, scale, s); break;
    case 8: launch_op_v<8>(v, op.n, sre, sim, ca, x, y, resid, scale, s); break;
    case 16: launch_op_v<16>(v, op.n, sre, sim, ca, x, y, resid, scale, s); break;
    default: launch_op_v<32>(v, op.n, sre, sim, ca, x, y, resid, scale, s); break;
  }
}

void launch_chain(const Chain& ch, const double* x, double* y, double* tmp, cudaStream_t s) {
  // out = P x, then out = Q_i out in append order (chain.cpp:117-126).
  const int L = ch.length();
  // Arrange ping-pong so that the last product lands in y.
  double* bufs[2] = {y, tmp};
  int cur = (L % 2 == 0) ? 0 : 1;
  launch_spmv(*ch.factors[0], x, bufs[cur], 1.0, s);
  for (int i = 1; i <= L; ++i) {
    launch_spmv(*ch.factors[size_t(i)], bufs[cur], bufs[cur ^ 1], 1.0, s);
    cur ^= 1;
  }
}

double device_norm2(int device, const double* x, int64_t n, cudaStream_t s) {
  DeviceGuard g(device);
  const int blocks = 256;
  DBuf<double> part(device, blocks + 1);
  k_sq_partial<<<blocks, 256, 0, s>>>(x, n, part.get());
  MPG_CHECK_LAUNCH();
  k_sum_partial<<<1, 32, 0, s>>>(part.get(), blocks, part.get() + blocks);
  MPG_CHECK_LAUNCH();
  count_launch(2);
  double h = 0.0;
  MPG_CUDA(cudaMemcpyAsync(&h, part.get() + blocks, sizeof(double), cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  return h;
}

CsrPtr op_explicit(const ShiftedOp& op, double sre, double sim, bool transpose) {
  auto& c = ctx(op.device);
  DeviceGuard g(op.device);
  const OpView v = op.view(transpose);
  const int n = int(op.n);
  const int pair = sim != 0.0;
  const int rows = pair ? 2 * n : n;
  DBuf<int> counts(op.device, size_t(rows) + 1), rp(op.device, size_t(rows) + 1);
  MPG_CUDA(cudaMemsetAsync(counts.get(), 0, (size_t(rows) + 1) * sizeof(int), c.stream));
  k_expl_count<<<grid_for(n), 256, 0, c.stream>>>(v.a, v.e, v.emode, pair, counts.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  exclusive_scan(op.device, counts.get(), rp.get(), rows, c.stream);
  int nnz = 0;
  MPG_CUDA(cudaMemcpyAsync(&nnz, rp.get() + rows, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  DBuf<int> ci(op.device, size_t(nnz));
  DBuf<double> val(op.device, size_t(nnz));
  k_expl_fill<<<grid_for(n), 256, 0, c.stream>>>(v.a, v.ae, v.ediag, v.emode, pair, sre, sim, rp.get(), ci.get(),
                                                 val.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return csr_from_device_parts(op.device, rows, rows, std::move(rp), std::move(ci), std::move(val));
}

}  // namespace mpg
