// Halo-staged sliced-ELL layout for the run-mode multi-RHS SpMVs (runtime.cuh
// HaloPattern). Built once per sparsity pattern, entirely on the device:
//   pass 1 (k_halo_count): per block of HALO_R rows, sort the block's column
//     indices in shared memory (bitonic), count the unique ones (the halo) and
//     the width of each 32-row slice;
//   host: prefix sums of the halo sizes and slice widths (one small copy);
//   pass 2 (k_halo_fill): sort again, write the halo, and for every entry its
//     16-bit local index (binary search in the block's halo) and its CSR
//     position (perm) in slice-column-major order; padding gets perm = -1.
// Values are then gathered through perm (k_halo_gather*), so a factor's values
// or an operator's (a, e) pairs share one pattern build.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "runtime.cuh"

namespace mpg {
namespace {

constexpr int HB_THREADS = 256;
constexpr int HB_SLICES = HALO_R / 32;

// Sort keys[0..P) ascending in shared memory (P a power of two <= HALO_MAXNZ).
__device__ void block_bitonic(int* keys, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
    }
  __syncthreads();
}

// Loads the block's columns, sorts them, compacts the unique ones into uniq
// (returns their count, or -1 if the block has too many entries).
__device__ int block_halo(const CsrView m, int r0, int r1, int* keys, int* uniq, int* scan) {
  const int nz0 = m.rowptr[r0], nz1 = m.rowptr[r1];
  const int cnt = nz1 - nz0;
  if (cnt > HALO_MAXNZ) return -1;
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) keys[i] = i < cnt ? m.colind[nz0 + i] : INT_MAX;
  block_bitonic(keys, P);
  // per-thread contiguous chunk: count heads, exclusive scan over threads, write
  const int per = (P + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(P, b + per);
  int c = 0;
  for (int i = b; i < e; ++i)
    if (keys[i] != INT_MAX && (i == 0 || keys[i] != keys[i - 1])) ++c;
  scan[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  int pos = scan[threadIdx.x] - c;
  for (int i = b; i < e; ++i)
    if (keys[i] != INT_MAX && (i == 0 || keys[i] != keys[i - 1])) uniq[pos++] = keys[i];
  const int total = scan[blockDim.x - 1];
  __syncthreads();
  return total;
}

constexpr size_t HB_SMEM = (2 * size_t(HALO_MAXNZ) + HB_THREADS) * sizeof(int);

__global__ void __launch_bounds__(HB_THREADS) k_halo_count(CsrView m, int* halo_cnt, int* slice_w) {
  extern __shared__ int hb_sm[];
  int *keys = hb_sm, *uniq = hb_sm + HALO_MAXNZ, *scan = hb_sm + 2 * HALO_MAXNZ;
  const int r0 = blockIdx.x * HALO_R, r1 = min(m.nrows, r0 + HALO_R);
  const int total = block_halo(m, r0, r1, keys, uniq, scan);
  if (threadIdx.x == 0) halo_cnt[blockIdx.x] = total;
  if (threadIdx.x < HB_SLICES) {
    int w = 0;
    for (int r = r0 + threadIdx.x * 32; r < min(r1, r0 + threadIdx.x * 32 + 32); ++r)
      w = max(w, m.rowptr[r + 1] - m.rowptr[r]);
    slice_w[blockIdx.x * HB_SLICES + threadIdx.x] = w;
  }
}

__global__ void __launch_bounds__(HB_THREADS) k_halo_fill(CsrView m, const int* hoff, const int* sptr, int* halo,
                                                          unsigned short* lidx, int* perm) {
  extern __shared__ int hb_sm[];
  int *keys = hb_sm, *uniq = hb_sm + HALO_MAXNZ, *scan = hb_sm + 2 * HALO_MAXNZ;
  const int r0 = blockIdx.x * HALO_R, r1 = min(m.nrows, r0 + HALO_R);
  const int total = block_halo(m, r0, r1, keys, uniq, scan);
  const int h0 = hoff[blockIdx.x];
  for (int i = threadIdx.x; i < total; i += blockDim.x) halo[h0 + i] = uniq[i];
  if (threadIdx.x >= HALO_R) return;
  const int row = r0 + threadIdx.x;
  const int slice = row >> 5, lane = row & 31;
  const int e0 = sptr[slice], w = (sptr[slice + 1] - e0) >> 5;
  int b = 0, len = 0;
  if (row < r1) {
    b = m.rowptr[row];
    len = m.rowptr[row + 1] - b;
  }
  for (int j = 0; j < w; ++j) {
    const int e = e0 + j * 32 + lane;
    if (j < len) {
      const int c = m.colind[b + j];
      int lo = 0, hi = total - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uniq[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      lidx[e] = static_cast<unsigned short>(lo);
      perm[e] = b + j;
    } else {
      lidx[e] = 0;
      perm[e] = -1;
    }
  }
}

__global__ void k_halo_gather(const int* perm, int64_t entries, const double* src, double* dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < entries; e += int64_t(gridDim.x) * blockDim.x) {
    const int p = perm[e];
    dst[e] = p >= 0 ? src[p] : 0.0;
  }
}

__global__ void k_halo_gather2(const int* perm, int64_t entries, const double2* src, double2* dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < entries; e += int64_t(gridDim.x) * blockDim.x) {
    const int p = perm[e];
    dst[e] = p >= 0 ? src[p] : make_double2(0.0, 0.0);
  }
}

// SELL-8: per 8-row slice the longest row (pass 1), then entries column-major
// within the slice (pass 2), padding with the row's own index and perm -1.
__global__ void k_sell8_width(CsrView m, int* w) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int r0 = s * 8;
  if (r0 >= m.nrows) return;
  int mx = 0;
  for (int r = r0; r < min(m.nrows, r0 + 8); ++r) mx = max(mx, m.rowptr[r + 1] - m.rowptr[r]);
  w[s] = mx;
}

__global__ void k_sell8_fill(CsrView m, const int* sptr, int* col, int* perm) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int nsl = (m.nrows + 7) / 8;
  if (row >= nsl * 8) return;
  const int s = row >> 3, r8 = row & 7;
  const int e0 = sptr[s], w = (sptr[s + 1] - e0) >> 3;
  int b = 0, len = 0;
  if (row < m.nrows) {
    b = m.rowptr[row];
    len = m.rowptr[row + 1] - b;
  }
  const int self = row < m.nrows ? row : 0;
  for (int j = 0; j < w; ++j) {
    const int e = e0 + 8 * j + r8;
    col[e] = j < len ? m.colind[b + j] : self;
    perm[e] = j < len ? b + j : -1;
  }
}

}  // namespace

Sell8Ptr sell8_build(const DevCsr& m) {
  if (m.nrows < 1 || m.nnz == 0) return nullptr;
  auto& c = ctx(m.device);
  DeviceGuard g(m.device);
  const int n = int(m.nrows);
  const int nsl = (n + 7) / 8;
  DBuf<int> w(m.device, size_t(nsl));
  k_sell8_width<<<(nsl + 255) / 256, 256, 0, c.stream>>>(m.view(), w.get());
  MPG_CHECK_LAUNCH();
  std::vector<int> hw(static_cast<size_t>(nsl));
  MPG_CUDA(cudaMemcpyAsync(hw.data(), w.get(), hw.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<int> sptr(static_cast<size_t>(nsl) + 1, 0);
  int64_t ent = 0;
  for (int s = 0; s < nsl; ++s) {
    ent += int64_t(hw[size_t(s)]) * 8;
    if (ent >= INT_MAX) return nullptr;
    sptr[size_t(s) + 1] = int(ent);
  }
  if (double(ent) > 1.25 * double(m.nnz) + 8.0 * nsl) return nullptr;
  auto p = std::make_shared<Sell8>();
  p->nrows = n;
  p->entries = ent;
  for (int s0 = 0; s0 < nsl; s0 += 8) p->max_tile = std::max(p->max_tile, sptr[size_t(std::min(nsl, s0 + 8))] - sptr[size_t(s0)]);
  p->sptr = DBuf<int>(m.device, sptr.size());
  p->col = DBuf<int>(m.device, size_t(std::max<int64_t>(1, ent)));
  p->perm = DBuf<int>(m.device, size_t(std::max<int64_t>(1, ent)));
  MPG_CUDA(cudaMemcpyAsync(p->sptr.get(), sptr.data(), sptr.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  k_sell8_fill<<<(nsl * 8 + 255) / 256, 256, 0, c.stream>>>(m.view(), p->sptr.get(), p->col.get(), p->perm.get());
  MPG_CHECK_LAUNCH();
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return p;
}

const Sell8* sell_of(const DevCsr& m, Sell8View* view) {
  std::scoped_lock l(m.mu);
  if (!m.sell_tried) {
    m.sell_tried = true;
    m.sell = sell8_build(m);
    if (m.sell) {
      auto& c = ctx(m.device);
      DeviceGuard g(m.device);
      m.sell_val = DBuf<double>(m.device, size_t(std::max<int64_t>(1, m.sell->entries)));
      k_halo_gather<<<std::max(1, c.sm_count * 8), 256, 0, c.stream>>>(m.sell->perm.get(), m.sell->entries,
                                                                       m.val.get(), m.sell_val.get());
      MPG_CHECK_LAUNCH();
    }
  }
  if (!m.sell) return nullptr;
  if (view) *view = Sell8View{m.sell->nrows, m.sell->sptr.get(), m.sell->col.get(), m.sell_val.get(), nullptr};
  return m.sell.get();
}

const Sell8* sell_of_op(const ShiftedOp& op, bool transpose, Sell8View* view) {
  const DevCsr& a = transpose ? *op.at : *op.a;
  Sell8View av{};
  const Sell8* p = sell_of(a, &av);
  if (!p) return nullptr;
  if (op.emode == E_SAMEPAT) {
    std::scoped_lock l(op.halo_mu);
    const int t = transpose ? 1 : 0;
    if (!op.sell_tried_op[t]) {
      op.sell_tried_op[t] = true;
      auto& c = ctx(op.device);
      DeviceGuard g(op.device);
      op.sell_ae[t] = DBuf<double2>(op.device, size_t(std::max<int64_t>(1, p->entries)));
      k_halo_gather2<<<std::max(1, c.sm_count * 8), 256, 0, c.stream>>>(
          p->perm.get(), p->entries, transpose ? op.ae_t.get() : op.ae.get(), op.sell_ae[t].get());
      MPG_CHECK_LAUNCH();
    }
    av.val2 = op.sell_ae[t].get();
  } else if (op.emode == E_GENERAL) {
    return nullptr;
  }
  if (view) *view = av;
  return p;
}

HaloPatternPtr halo_pattern_build(const DevCsr& m) {
  if (m.nrows < 1 || m.nrows != m.ncols || m.nnz == 0) return nullptr;
  auto& c = ctx(m.device);
  DeviceGuard g(m.device);
  const int n = int(m.nrows);
  const int nblocks = (n + HALO_R - 1) / HALO_R;
  const int nslices = nblocks * (HALO_R / 32);
  DBuf<int> cnt(m.device, size_t(nblocks)), widths(m.device, size_t(nslices));
  cudaFuncSetAttribute(k_halo_count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(HB_SMEM));
  cudaFuncSetAttribute(k_halo_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, int(HB_SMEM));
  k_halo_count<<<nblocks, HB_THREADS, HB_SMEM, c.stream>>>(m.view(), cnt.get(), widths.get());
  MPG_CHECK_LAUNCH();
  std::vector<int> hc(static_cast<size_t>(nblocks));
  std::vector<int> hw(static_cast<size_t>(nslices));
  MPG_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), hc.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaMemcpyAsync(hw.data(), widths.get(), hw.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  auto p = std::make_shared<HaloPattern>();
  std::vector<int> hoff(static_cast<size_t>(nblocks) + 1, 0);
  std::vector<int> sptr(static_cast<size_t>(nslices) + 1, 0);
  if (std::getenv("MPG_HALO_DEBUG")) {
    int mx = 0, bad = 0;
    double sum = 0.0;
    for (int v : hc) {
      mx = std::max(mx, v);
      bad += v < 0 || v > HALO_MAX;
      sum += v;
    }
    std::fprintf(stderr, "[halo] n=%d nnz=%lld blocks=%d max_halo=%d mean_halo=%.1f over_limit=%d\n", n,
                 (long long)m.nnz, nblocks, mx, sum / nblocks, bad);
  }
  for (int b = 0; b < nblocks; ++b) {
    if (hc[size_t(b)] < 0 || hc[size_t(b)] > HALO_MAX) return nullptr;
    hoff[size_t(b) + 1] = hoff[size_t(b)] + hc[size_t(b)];
    p->max_halo = std::max(p->max_halo, hc[size_t(b)]);
  }
  int64_t ent = 0;
  for (int s = 0; s < nslices; ++s) {
    ent += int64_t(hw[size_t(s)]) * 32;
    if (ent >= INT_MAX) return nullptr;
    sptr[size_t(s) + 1] = int(ent);
  }
  // the padding must stay small: the SpMV streams every padded entry
  if (double(ent) > 1.25 * double(m.nnz) + 32.0 * nslices) return nullptr;
  p->nrows = n;
  p->nblocks = nblocks;
  p->entries = ent;
  p->hoff = DBuf<int>(m.device, hoff.size());
  p->sptr = DBuf<int>(m.device, sptr.size());
  p->halo = DBuf<int>(m.device, size_t(std::max(1, hoff.back())));
  p->perm = DBuf<int>(m.device, size_t(std::max<int64_t>(1, ent)));
  p->lidx = DBuf<unsigned short>(m.device, size_t(std::max<int64_t>(1, ent)));
  MPG_CUDA(cudaMemcpyAsync(p->hoff.get(), hoff.data(), hoff.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  MPG_CUDA(cudaMemcpyAsync(p->sptr.get(), sptr.data(), sptr.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  k_halo_fill<<<nblocks, HB_THREADS, HB_SMEM, c.stream>>>(m.view(), p->hoff.get(), p->sptr.get(), p->halo.get(),
                                                    p->lidx.get(), p->perm.get());
  MPG_CHECK_LAUNCH();
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return p;
}

const HaloPattern* halo_of(const DevCsr& m, HaloView* view) {
  std::scoped_lock l(m.mu);
  if (!m.halo_tried) {
    m.halo_tried = true;
    m.halo = halo_pattern_build(m);
    if (m.halo) {
      auto& c = ctx(m.device);
      DeviceGuard g(m.device);
      m.halo_val = DBuf<double>(m.device, size_t(std::max<int64_t>(1, m.halo->entries)));
      k_halo_gather<<<std::max(1, c.sm_count * 8), 256, 0, c.stream>>>(m.halo->perm.get(), m.halo->entries,
                                                                       m.val.get(), m.halo_val.get());
      MPG_CHECK_LAUNCH();
    }
  }
  if (!m.halo) return nullptr;
  if (view) {
    const HaloPattern& p = *m.halo;
    *view = HaloView{p.nrows, p.hoff.get(), p.halo.get(), p.sptr.get(), p.lidx.get(), m.halo_val.get(), nullptr};
  }
  return m.halo.get();
}

const HaloPattern* halo_of_op(const ShiftedOp& op, bool transpose, HaloView* view) {
  const DevCsr& a = transpose ? *op.at : *op.a;
  HaloView av{};
  const HaloPattern* p = halo_of(a, &av);
  if (!p) return nullptr;
  if (op.emode == E_SAMEPAT) {
    std::scoped_lock l(op.halo_mu);
    const int t = transpose ? 1 : 0;
    if (!op.halo_tried[t]) {
      op.halo_tried[t] = true;
      auto& c = ctx(op.device);
      DeviceGuard g(op.device);
      op.halo_ae[t] = DBuf<double2>(op.device, size_t(std::max<int64_t>(1, p->entries)));
      k_halo_gather2<<<std::max(1, c.sm_count * 8), 256, 0, c.stream>>>(
          p->perm.get(), p->entries, transpose ? op.ae_t.get() : op.ae.get(), op.halo_ae[t].get());
      MPG_CHECK_LAUNCH();
    }
    av.val2 = op.halo_ae[t].get();
  } else if (op.emode == E_GENERAL) {
    return nullptr;
  }
  if (view) *view = av;
  return p;
}

}  // namespace mpg
