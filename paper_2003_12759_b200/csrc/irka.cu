// IRKA driver (BIRKA with N = 0, proj/src/birka.cpp:139-310), generalised to
// a mass matrix E, plus the shift-sweep benchmark (run_spai_bench,
// proj/src/bench.cpp:159-249).
//
// Per sweep: real block spectrum of K_r on the host (r x r), right-hand
// sides B f2 / C c2 on the device, one GMRES per shift unit and side (the
// reference's joint n*r solve is block diagonal for N = 0, so the units are
// independent), all advanced together by gmres_batch;
// V, W by CholQR2 (K5: tall-skinny Gram + small triangular apply), the
// projection E_r = W^T E V, A_r = W^T A V, K_r = E_r^{-1} A_r,
// f_r = E_r^{-1} W^T B, c_r = V^T C; convergence on the sorted spectrum.
// With E = I this is the reference's update (E_r = W^T V).
//
// Multi-GPU: (side, unit) solves are sharded by a static slot -> rank map so
// each preconditioner chain stays on its rank; the only exchange is the
// all-gather of the solved V/W columns (K6), after which every rank projects
// redundantly.
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <limits>
#include <random>

#include "host/small_dense.hpp"
#include "host/h2.hpp"
#include "irka.hpp"

namespace mpg {
namespace {

using host::Mat;

// rows per tile of k_ts_gram: as many as 48 KB of shared memory holds (multiple of 64, at most 512)
__host__ __device__ __forceinline__ int ts_rows(int a, int b) {
  int ch = (47 * 1024 / 8) / (a + b) - 1;
  ch = ch > 512 ? 512 : ch;
  return ch < 64 ? 64 : ch & ~63;
}

// part[blk][i + a*j] = sum over this block's rows of X[row, i] * Y[row, j]
__global__ void __launch_bounds__(256) k_ts_gram(const double* __restrict__ X, int64_t ldx, int a,
                                                 const double* __restrict__ Y, int64_t ldy, int b, int64_t n,
                                                 double* __restrict__ part) {
  extern __shared__ double sm[];
  const int CH = ts_rows(a, b);
  const int LD = CH + 1;     // padded row stride of a column tile (bank spread)
  double* xs = sm;           // LD * a
  double* ys = sm + LD * a;  // LD * b
  const int npair = a * b;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = int64_t(blockIdx.x) * CH; r0 < n; r0 += int64_t(gridDim.x) * CH) {
    const int rows = n - r0 < CH ? int(n - r0) : CH;
    __syncthreads();
    for (int t = threadIdx.x; t < CH * a; t += blockDim.x) {
      const int i = t / CH, r = t % CH;
      xs[i * LD + r] = r < rows ? X[r0 + r + ldx * i] : 0.0;
    }
    for (int t = threadIdx.x; t < CH * b; t += blockDim.x) {
      const int j = t / CH, r = t % CH;
      ys[j * LD + r] = r < rows ? Y[r0 + r + ldy * j] : 0.0;
    }
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
      const int pidx = threadIdx.x + q * blockDim.x;
      if (pidx >= npair) break;
      const int i = pidx % a, j = pidx / a;
      double s = acc[q];
      for (int r = 0; r < CH; ++r) s = fma(xs[i * LD + r], ys[j * LD + r], s);
      acc[q] = s;
    }
  }
  for (int q = 0; q < 4; ++q) {
    const int pidx = threadIdx.x + q * blockDim.x;
    if (pidx < npair) part[size_t(blockIdx.x) * npair + pidx] = acc[q];
  }
}

// Y[:, j] = sum_i X[:, i] M[i, j]   (M is a x b, column-major, in global memory)
__global__ void __launch_bounds__(256) k_ts_apply(const double* __restrict__ X, int64_t ldx, int a,
                                                  const double* __restrict__ M, int b, double* __restrict__ Y,
                                                  int64_t ldy, int64_t n) {
  extern __shared__ double ms[];
  for (int t = threadIdx.x; t < a * b; t += blockDim.x) ms[t] = M[t];
  __syncthreads();
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
    double xr[64];
    for (int i = 0; i < a; ++i) xr[i] = X[r + ldx * i];
    for (int j = 0; j < b; ++j) {
      double s = 0.0;
      for (int i = 0; i < a; ++i) s = fma(xr[i], ms[i + a * j], s);
      Y[r + ldy * j] = s;
    }
  }
}

Mat ts_gram(int dev, const double* X, int64_t ldx, int a, const double* Y, int64_t ldy, int b, int64_t n) {
  if (a > 1024) throw std::invalid_argument("ts_gram: at most 1024 rows in the Gram");
  if (a * b > 1024) {  // tile over column blocks of Y (one launch holds <= 1024 products per CTA)
    const int bw = 1024 / a;
    Mat out(a, b);
    for (int j0 = 0; j0 < b; j0 += bw) {
      const int w = std::min(bw, b - j0);
      const Mat blk = ts_gram(dev, X, ldx, a, Y + size_t(ldy) * j0, ldy, w, n);
      for (int j = 0; j < w; ++j)
        for (int i = 0; i < a; ++i) out(i, j0 + j) = blk(i, j);
    }
    return out;
  }
  auto& c = ctx(dev);
  const int ch = ts_rows(a, b);
  const int blocks = std::max(1, std::min<int>(c.sm_count * 4, int((n + ch - 1) / ch)));
  DBuf<double> part(dev, size_t(blocks) * size_t(a) * size_t(b));
  const size_t smem = size_t(ch + 1) * size_t(a + b) * sizeof(double);
  k_ts_gram<<<blocks, 256, smem, c.stream>>>(X, ldx, a, Y, ldy, b, n, part.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  std::vector<double> h(part.n);
  MPG_CUDA(cudaMemcpyAsync(h.data(), part.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  Mat out(a, b);
  for (int blk = 0; blk < blocks; ++blk)
    for (int p = 0; p < a * b; ++p) out.a[size_t(p)] += h[size_t(blk) * size_t(a * b) + size_t(p)];
  return out;
}

void ts_apply(int dev, const double* X, int64_t ldx, int a, const Mat& M, double* Y, int64_t ldy, int64_t n) {
  auto& c = ctx(dev);
  if (a > 64) throw std::invalid_argument("ts_apply: at most 64 columns");
  DBuf<double> dm(dev, M.a.size());
  MPG_CUDA(cudaMemcpyAsync(dm.get(), M.a.data(), M.a.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  const int blocks = std::max(1, std::min<int>(c.sm_count * 8, int((n + 255) / 256)));
  k_ts_apply<<<blocks, 256, M.a.size() * sizeof(double), c.stream>>>(X, ldx, a, dm.get(), M.cols, Y, ldy, n);
  MPG_CHECK_LAUNCH();
  count_launch();
  MPG_CUDA(cudaStreamSynchronize(c.stream));
}

// CholQR2 in place on X (n x r, ld = n); returns false if X is rank deficient.
bool cholqr2(int dev, double* X, int64_t n, int r) {
  DBuf<double> tmp(dev, size_t(n) * size_t(r));
  for (int pass = 0; pass < 2; ++pass) {
    const Mat g = ts_gram(dev, X, n, r, X, n, r, n);
    Mat R;
    if (!host::cholesky_upper(g, R)) return false;
    // reject a numerically rank-deficient block (Cholesky of the Gram squares kappa)
    double dmax = 0.0, dmin = 1e300;
    for (int i = 0; i < r; ++i) { dmax = std::max(dmax, R(i, i)); dmin = std::min(dmin, R(i, i)); }
    if (pass == 0 && dmin < 1e-7 * dmax) return false;
    ts_apply(dev, X, n, r, host::upper_inverse(R), tmp.get(), n, n);
    MPG_CUDA(cudaMemcpyAsync(X, tmp.get(), size_t(n) * size_t(r) * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx(dev).stream));
  }
  MPG_CUDA(cudaStreamSynchronize(ctx(dev).stream));
  return true;
}

void orthonormalize(int dev, double* X, int64_t n, int r) {
  if (cholqr2(dev, X, n, r)) return;
  // Host Householder fallback (thin_q, birka.cpp:125-128) for ill-conditioned blocks.
  auto& c = ctx(dev);
  Mat h(int(n), r);
  MPG_CUDA(cudaMemcpyAsync(h.a.data(), X, h.a.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  Mat q = host::householder_q(h);
  MPG_CUDA(cudaMemcpyAsync(X, q.a.data(), q.a.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
}

// Blocks of 32 unit columns, row-major [n][32] (lane = column): one launch per
// chain factor / operator / residual per block instead of one sync per column.
__global__ void k_unit_block(double* x, int64_t n, int64_t j0) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n * 32; t += int64_t(gridDim.x) * blockDim.x)
    x[t] = (t / 32 == j0 + (t & 31)) ? 1.0 : 0.0;
}
__global__ void k_spmm32(CsrView a, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; row < a.nrows;
       row += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int k = a.rowptr[row]; k < a.rowptr[row + 1]; ++k) acc += a.val[k] * x[int64_t(a.colind[k]) * 32 + lane];
    y[row * 32 + lane] = acc;
  }
}
__global__ void k_resid_block(const double* __restrict__ y, int64_t n, int64_t j0, int valid, double* acc) {
  double sq = 0.0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n * 32; t += int64_t(gridDim.x) * blockDim.x) {
    const int l = int(t & 31);
    if (l >= valid) continue;
    const double d = y[t] - ((t / 32 == j0 + l) ? 1.0 : 0.0);
    sq += d * d;
  }
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(acc, t);
  }
}

double std_residual(const CsrPtr& m, const ChainPtr& ch) {
  // ||I - M P||_F / sqrt(n) (chain.cpp:140-157)
  const int dev = m->device;
  auto& c = ctx(dev);
  const int64_t n = m->nrows;
  if (n == 0) return 0.0;
  DBuf<double> e(dev, size_t(n) * 32), b0(dev, size_t(n) * 32), b1(dev, size_t(n) * 32), acc(dev, 1);
  MPG_CUDA(cudaMemsetAsync(acc.get(), 0, sizeof(double), c.stream));
  const int grid = int(std::min<int64_t>((n * 32 + 255) / 256, 148 * 8));
  const int L = ch->length();
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    k_unit_block<<<grid, 256, 0, c.stream>>>(e.get(), n, j0);
    MPG_CHECK_LAUNCH();
    double* bufs[2] = {b0.get(), b1.get()};
    int cur = 0;
    k_spmm32<<<grid, 256, 0, c.stream>>>(ch->factors[0]->view(), e.get(), bufs[cur]);
    MPG_CHECK_LAUNCH();
    for (int i = 1; i <= L; ++i, cur ^= 1) {
      k_spmm32<<<grid, 256, 0, c.stream>>>(ch->factors[size_t(i)]->view(), bufs[cur], bufs[cur ^ 1]);
      MPG_CHECK_LAUNCH();
    }
    k_spmm32<<<grid, 256, 0, c.stream>>>(m->view(), bufs[cur], e.get());
    MPG_CHECK_LAUNCH();
    k_resid_block<<<grid, 256, 0, c.stream>>>(e.get(), n, j0, int(std::min<int64_t>(32, n - j0)), acc.get());
    MPG_CHECK_LAUNCH();
    count_launch(L + 4);
  }
  double sq = 0.0;
  MPG_CUDA(cudaMemcpyAsync(&sq, acc.get(), sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  MPG_CUDA(cudaStreamSynchronize(c.stream));
  return std::sqrt(std::max(sq, 0.0)) / std::sqrt(double(n));
}

}  // namespace

double std_residual_public(const CsrPtr& m, const ChainPtr& ch) { return std_residual(m, ch); }

// IRKA's projection step (birka.cpp:283-291, E-generalised): E_r = W^T E V,
// A_r = W^T A V for device or host V, W (n x r, column-major); r <= 32.
void project_public(const ShiftedOp& op, const double* v_any, const double* w_any, int r, Mat& er, Mat& ar) {
  const int dev = op.device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = op.n;
  if (r < 1 || r > 32) throw std::invalid_argument("project: 1 <= r <= 32");
  DBuf<double> V(dev, size_t(n) * r), W(dev, size_t(n) * r), AV(dev, size_t(n) * r), EV(dev, size_t(n) * r);
  copy_in(V.get(), v_any, size_t(n) * r, s);
  copy_in(W.get(), w_any, size_t(n) * r, s);
  for (int j = 0; j < r; ++j) {
    launch_spmv(*op.a, V.get() + size_t(n) * j, AV.get() + size_t(n) * j, 1.0, s);
    launch_op(op, false, 1.0, 0.0, 0.0, V.get() + size_t(n) * j, EV.get() + size_t(n) * j, nullptr, 1.0, s, nullptr);
    count_launch(2);
  }
  er = ts_gram(dev, W.get(), n, r, EV.get(), n, r, n);
  ar = ts_gram(dev, W.get(), n, r, AV.get(), n, r, n);
}

namespace {

struct SlotPrecond {
  ChainPtr chain;
  CsrPtr prev_explicit;
  int width = 0;
};

// birka_default_seed (birka.cpp:41-89): 20 power iterations of K on the device for the spectral radius
// (skipped when init_shifts are given), then fr and cr from the same mt19937_64 stream.
void default_seed(const DevCsr& a, const IrkaSettings& cfg, Mat& kr, Mat& fr, Mat& cr, cudaStream_t s) {
  const int dev = a.device;
  const int64_t n = a.nrows;
  const int r = cfg.r;
  std::mt19937_64 rng(cfg.seed);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  std::vector<double> x(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) x[size_t(i)] = unit(rng);
  if (cfg.init_shifts.empty()) {
    double radius = 0.0, xn = 0.0;
    for (double v : x) xn += v * v;
    xn = std::sqrt(xn);
    if (xn > 0.0) {
      for (double& v : x) v /= xn;
      DBuf<double> dx(dev, size_t(n)), dy(dev, size_t(n));
      copy_in(dx.get(), x.data(), size_t(n), s);
      for (int it = 0; it < 20; ++it) {
        launch_spmv(a, dx.get(), dy.get(), 1.0, s);
        const double ny = std::sqrt(device_norm2(dev, dy.get(), n, s));
        if (ny == 0.0) { radius = 0.0; break; }
        radius = ny;
        std::vector<double> hy(static_cast<size_t>(n));
        MPG_CUDA(cudaMemcpyAsync(hy.data(), dy.get(), size_t(n) * 8, cudaMemcpyDeviceToHost, s));
        MPG_CUDA(cudaStreamSynchronize(s));
        for (double& v : hy) v /= ny;
        copy_in(dx.get(), hy.data(), size_t(n), s);
      }
    }
    if (!(radius > 0.0) || !std::isfinite(radius)) radius = 1.0;
    for (int i = 0; i < r; ++i) {
      const double t = r == 1 ? 1.0 : double(i) / (r - 1);
      kr(i, i) = -radius * std::pow(10.0, -3.0 * (1.0 - t));
    }
  } else {
    if (int(cfg.init_shifts.size()) != r) throw ConfigError("irka: init_shifts must have r entries");
    for (int i = 0; i < r; ++i) kr(i, i) = -cfg.init_shifts[size_t(i)];
  }
  for (Mat* mm : {&fr, &cr})
    for (int j = 0; j < mm->cols; ++j) {
      double nn = 0.0;
      for (int i = 0; i < r; ++i) { (*mm)(i, j) = unit(rng); nn += (*mm)(i, j) * (*mm)(i, j); }
      nn = std::sqrt(nn);
      if (nn > 0.0)
        for (int i = 0; i < r; ++i) (*mm)(i, j) /= nn;
    }
}

}  // namespace

double shard_cost(int width, int last_iterations) {
  const double k = last_iterations < 0 ? 100.0 : double(std::max(last_iterations, 1));
  return double(width) * k * (k + 40.0);
}

std::vector<int> shard_plan(const std::vector<double>& cost, const std::vector<int>& fixed, int world) {
  if (world < 1) throw std::invalid_argument("shard_plan: world must be at least 1");
  if (fixed.size() != cost.size()) throw std::invalid_argument("shard_plan: cost and fixed differ in length");
  std::vector<int> owner(cost.size(), 0);
  std::vector<double> load(size_t(world), 0.0);
  std::vector<size_t> free_units;
  for (size_t i = 0; i < cost.size(); ++i) {
    if (fixed[i] >= world) throw std::invalid_argument("shard_plan: fixed owner out of range");
    if (fixed[i] >= 0) {
      owner[i] = fixed[i];
      load[size_t(fixed[i])] += cost[i];
    } else {
      free_units.push_back(i);
    }
  }
  std::stable_sort(free_units.begin(), free_units.end(), [&](size_t x, size_t y) { return cost[x] > cost[y]; });
  for (size_t i : free_units) {
    const int o = int(std::min_element(load.begin(), load.end()) - load.begin());
    owner[i] = o;
    load[size_t(o)] += cost[i];
  }
  return owner;
}

IrkaResult irka_run(const ShiftedOp& op, const double* b_any, int m, const double* c_any, int q, const IrkaSettings& cfg,
                    int rank, int world, mpg_allgather_fn allgather, void* agctx) {
  const int dev = op.device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = op.n;
  const int r = cfg.r;
  if (m < 1 || q < 1) throw ConfigError("irka: B and C need at least one column");
  if (cfg.max_sweeps < 1) throw ConfigError("birka: max_sweeps must be at least 1");
  if (cfg.max_chain_len < 1) throw ConfigError("birka: max_chain_len must be at least 1");
  if (r < 1) throw ConfigError("birka: reduced order must be at least 1");
  if (int64_t(r) > n) throw ConfigError("birka: reduced order exceeds the system dimension");
  if (r > 64 || m > 64 || q > 64) throw ConfigError("irka: r, m, q are limited to 64 on the GPU path");
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("irka: bad rank/world");
  if (world > 1 && !allgather) throw std::invalid_argument("irka: world > 1 needs an allgather callback");

  DBuf<double> B(dev, size_t(n) * m), C(dev, size_t(n) * q);
  copy_in(B.get(), b_any, size_t(n) * m, s);
  copy_in(C.get(), c_any, size_t(n) * q, s);

  Mat kr(r, r), fr(r, m), cr(r, q);
  default_seed(*op.a, cfg, kr, fr, cr, s);
  {  // a caller-supplied initial state replaces the seed part by part (birka.cpp:145)
    auto take = [](Mat& dst, const std::vector<double>& src, const char* what) {
      if (src.empty()) return;
      if (src.size() != dst.a.size()) throw ConfigError(std::string("birka: initial state dimensions do not match the system (") + what + ")");
      dst.a = src;
    };
    take(kr, cfg.init_kr, "kr");
    take(fr, cfg.init_fr, "fr");
    take(cr, cfg.init_cr, "cr");
  }

  IrkaResult res;
  res.reduced_order = r;
  DBuf<double> X(dev, size_t(n) * r), Y(dev, size_t(n) * r), RHS(dev, size_t(n) * r * 2);
  DBuf<double> AV(dev, size_t(n) * r), EV(dev, size_t(n) * r);
  std::map<std::pair<int, int>, SlotPrecond> slots;   // (side, first column)
  std::map<std::pair<int, int>, ChainPtr> frozen;      // (side, unit width) -> frozen base
  std::map<std::pair<int, int>, std::pair<int, int>> slot_owner;  // (side, c0) -> (rank, width)
  std::map<std::pair<int, int>, int> slot_iters;                  // (side, c0) -> last sweep's iterations
  std::mt19937_64 perturb_rng(cfg.seed ^ 0x9e3779b97f4a7c15ull);
  std::vector<host::Eig> lambda_prev = host::sorted_eigenvalues(kr);
  bool converged = false;
  int sweeps_done = 0;
  const GmresOptions gopt = cfg.gmres;

  int last_max_its = 0;
  const bool timing = std::getenv("MPG_IRKA_TIMING") != nullptr;
  auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  for (int z = 1; z <= cfg.max_sweeps && !converged; ++z) {
    const double tz0 = wall();
    double t_build = 0.0, t_gmres = 0.0;
    host::Spectrum spec;
    if (!host::real_spectrum(kr, spec)) {  // birka.cpp:167-180
      std::uniform_real_distribution<double> unit(-1.0, 1.0);
      Mat nudged = kr;
      const double scale = 1e-8 * std::max(1.0, host::fro(kr));
      for (double& v : nudged.a) v += scale * unit(perturb_rng);
      if (!host::real_spectrum(nudged, spec))
        throw SolverError("birka: reduced state matrix is not diagonalizable (sweep " + std::to_string(z) +
                          "), even after perturbation");
      kr = nudged;
      lambda_prev = host::sorted_eigenvalues(kr);
    }
    if (cfg.mirror_unstable) {
      // Standard IRKA safeguard (not in the reference): reflect unstable
      // reduced poles, Re(lambda) -> -|Re(lambda)|, so every shift sigma = -lambda
      // has a positive real part.
      for (int i = 0; i < r; ++i)
        if (spec.blocks(i, i) > 0.0) spec.blocks(i, i) = -spec.blocks(i, i);
    }
    // birka.cpp:182-183: f2 = fr^T R^{-T} (m x r), c2 = cr^T R (q x r); the
    // trial right-hand sides are B f2 and the test ones C c2 (:199).
    const Mat f2t = host::mul(spec.basis_inv, fr);                   // (f2)^T = R^{-1} fr   (r x m)
    const Mat c2t = host::mul(host::transpose(spec.basis), cr);      // (c2)^T = R^T cr      (r x q)
    // right-hand sides: side 0 columns B f2 -> RHS[:, 0..r), side 1 C c2 -> RHS[:, r..2r)
    ts_apply(dev, B.get(), n, m, host::transpose(f2t), RHS.get(), n, n);
    ts_apply(dev, C.get(), n, q, host::transpose(c2t), RHS.get() + size_t(n) * r, n, n);
    for (int side = 0; side < 2; ++side) {
      const double bn = device_norm2(dev, RHS.get() + size_t(n) * r * side, n * r, s);
      if (bn == 0.0)
        throw SolverError(std::string("birka: zero right-hand side on the ") + (side == 0 ? "trial" : "test") +
                          " side (sweep " + std::to_string(z) + "); input/output maps must be nonzero");
    }
    // ---- solve tasks for this rank ----
    struct Task { int side, c0, w; double sre, sim; int owner; };
    std::vector<Task> mine, all;
    for (int side = 0; side < 2; ++side)
      for (size_t u = 0; u < spec.unit_start.size(); ++u) {
        const int c0 = spec.unit_start[u], w = spec.unit_width[u];
        all.push_back(Task{side, c0, w, -spec.blocks(c0, c0), w == 2 ? -spec.blocks(c0, c0 + 1) : 0.0, 0});
      }
    {
      // Owner map, identical on every rank (it depends only on data all ranks
      // share): units are placed longest-first on the least-loaded rank, with
      // the cost of a solve modelled from the previous sweep's iterations of
      // its slot (w K (K + 40): the Gram-Schmidt work grows as K^2). In the
      // chain-bearing modes a slot keeps its rank while its shape is
      // unchanged, so its vertical chain stays local.
      const bool sticky = cfg.mode == MPG_PRECOND_REUSE_CHAIN;
      std::vector<double> cost(all.size());
      std::vector<int> fixed(all.size(), -1);
      for (size_t i = 0; i < all.size(); ++i) {
        auto it = slot_iters.find({all[i].side, all[i].c0});
        cost[i] = shard_cost(all[i].w, it == slot_iters.end() ? -1 : it->second);
        auto ot = slot_owner.find({all[i].side, all[i].c0});
        if (sticky && ot != slot_owner.end() && ot->second.second == all[i].w) fixed[i] = ot->second.first;
      }
      const std::vector<int> owner = shard_plan(cost, fixed, world);
      for (size_t i = 0; i < all.size(); ++i) {
        all[i].owner = owner[i];
        slot_owner[{all[i].side, all[i].c0}] = {owner[i], all[i].w};
      }
      for (const Task& t : all)
        if (t.owner == rank) mine.push_back(t);
    }
    std::vector<SolveSpec> specs;
    std::vector<mpg_report_row> rows;
    DBuf<double> SOL(dev, size_t(n) * r * 2);
    for (const Task& t : mine) {
      mpg_report_row row{};
      row.sweep = z;
      row.point = t.side + 1;
      row.kind = MPG_KIND_NONE;
      row.min_residual = row.matrix_change = row.standard_residual = std::nan("");
      ChainPtr chain;
      if (cfg.mode != MPG_PRECOND_NONE) {
        const auto key = std::make_pair(t.side, t.c0);
        const bool tr = t.side == 1;
        if (cfg.mode == MPG_PRECOND_REUSE_FROZEN) {
          auto fk = std::make_pair(t.side, t.w);
          auto it = frozen.find(fk);
          if (it == frozen.end() && t.w == 2 && frozen.count({t.side, 1})) {
            chain = frozen[{t.side, 1}];  // n x n base applied blockwise on the pair
            row.kind = MPG_KIND_REUSED_SAME_MATRIX;
          } else if (it == frozen.end()) {
            CsrPtr M = op_explicit(op, t.sre, t.sim, tr);
            SpaiOutcome so = spai_or_update(M, nullptr, cfg.spai, false);
            auto ch = std::make_shared<Chain>();
            ch->factors.push_back(so.p);
            chain = ch;
            frozen[fk] = chain;
            row.kind = MPG_KIND_FRESH;
            row.build_seconds = so.build_seconds;
            if (M->nrows <= cfg.standard_residual_max_dim) row.standard_residual = std_residual(M, chain);
          } else {
            chain = it->second;
            row.kind = MPG_KIND_REUSED_SAME_MATRIX;
          }
        } else {
          CsrPtr M = op_explicit(op, t.sre, t.sim, tr);
          SlotPrecond& sp = slots[key];
          if (sp.width != t.w) sp = SlotPrecond{nullptr, nullptr, t.w};
          if (cfg.mode == MPG_PRECOND_FRESH || !sp.chain || sp.chain->length() + 1 > cfg.max_chain_len) {
            SpaiOutcome so = spai_or_update(M, nullptr, cfg.spai, false);
            auto ch = std::make_shared<Chain>();
            ch->factors.push_back(so.p);
            sp.chain = ch;
            row.kind = MPG_KIND_FRESH;
            row.build_seconds = so.build_seconds;
          } else {
            SpaiOutcome so = spai_or_update(M, sp.prev_explicit, cfg.spai, false);
            auto ch = std::make_shared<Chain>(*sp.chain);
            ch->factors.push_back(so.p);
            sp.chain = ch;
            row.kind = MPG_KIND_VERTICAL;
            row.build_seconds = so.build_seconds;
            row.min_residual = so.min_residual;
            row.matrix_change = so.matrix_change;
          }
          if (cfg.mode == MPG_PRECOND_REUSE_CHAIN) sp.prev_explicit = M;
          chain = sp.chain;
          if (M->nrows <= cfg.standard_residual_max_dim) row.standard_residual = std_residual(M, chain);
        }
      }
      SolveSpec sp;
      sp.sre = t.sre;
      sp.sim = t.sim;
      sp.transpose = t.side == 1;
      sp.chain = chain;
      sp.b = RHS.get() + size_t(n) * (size_t(r) * t.side + t.c0);
      sp.x = SOL.get() + size_t(n) * (size_t(r) * t.side + t.c0);
      specs.push_back(sp);
      rows.push_back(row);
    }
    // batches bounded by device memory (each solve may grow to max_iter + 2 basis vectors)
    size_t free_b = 0, total_b = 0;
    MPG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    cudaMemPool_t pool;
    MPG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    const double avail = double(free_b) + double(reserved - used);
    // Basis panels are allocated as a solve grows, so a batch is sized by the
    // iterations the solves are expected to take (1.5x the previous sweep's
    // longest solve, 600 for the first sweep), not by max_iter.
    const int est_its = std::min(gopt.max_iter, z == 1 ? 600 : std::max(128, int(1.5 * double(last_max_its))));
    // at most 16 solves per batch (memory permitting): both sides of a sweep advance together, so the
    // per-iteration fixed costs (control kernels, idle launches, kernel tails) are paid once and every
    // side's reals and pairs share their 8-column groups. Round 1 measured batches of 7-8 faster by 4 %;
    // with the round-2 kernels the C3 IRKA runs 1.10 s per sweep at 16 against 1.17 s at 8.
    const int max_batch = std::getenv("MPG_IRKA_MAXBATCH") ? std::max(1, std::atoi(std::getenv("MPG_IRKA_MAXBATCH"))) : 16;
    std::vector<size_t> bounds{0};
    {
      double acc = 0.0;
      for (size_t i = 0; i < specs.size(); ++i) {
        const double ns_i = specs[i].sim != 0.0 ? 2.0 * double(n) : double(n);
        const double need = 12.0 * (ns_i + 64.0) * double(est_its + 72) + 1e7;  // fp64 basis + its float shadow
        if (i > bounds.back() && (acc + need > 0.85 * avail || int(i - bounds.back()) >= max_batch)) {
          bounds.push_back(i);
          acc = 0.0;
        }
        acc += need;
      }
      bounds.push_back(specs.size());
    }
    int sweep_max_its = 0;
    struct Failure { bool failed; int side, c0; double rel; int its; } fail{false, 0, 0, 0.0, 0};
    std::vector<int> its_mine(mine.size(), 0);
    t_build = wall() - tz0;
    for (size_t bi = 0; bi + 1 < bounds.size(); ++bi) {
      const size_t b0 = bounds[bi];
      std::vector<SolveSpec> batch(specs.begin() + long(b0), specs.begin() + long(bounds[bi + 1]));
      const double tg0 = wall();
      std::vector<GmresOutcome> outc = gmres_batch(op, batch, gopt);
      t_gmres += wall() - tg0;
      for (const GmresOutcome& o : outc) sweep_max_its = std::max(sweep_max_its, o.iterations);
      for (size_t i = 0; i < outc.size(); ++i) {
        mpg_report_row& row = rows[b0 + i];
        row.solves = 1;
        row.iterations = outc[i].iterations;
        row.gmres_seconds = outc[i].solve_seconds;
        res.total_iterations += outc[i].iterations;
        ++res.total_solves;
        its_mine[b0 + i] = outc[i].iterations;
        if (!outc[i].converged && !fail.failed) {
          const Task& t = mine[b0 + i];
          fail = Failure{true, t.side, t.c0, outc[i].final_residual / std::max(outc[i].rhs_norm, 1e-300),
                         outc[i].iterations};
        }
      }
      if (fail.failed && world == 1) break;
    }
    res.rows.insert(res.rows.end(), rows.begin(), rows.end());
    last_max_its = std::max(last_max_its == 0 ? 0 : last_max_its / 2, sweep_max_its);
    // ---- exchange (K6): all-gather the solved columns ----
    // Each rank's block is its solved columns followed by a status header
    // (failure flag and coordinates, then the iterations of its units), so a
    // solve that fails on one rank is raised on every rank after the
    // exchange instead of leaving the others blocked in the collective, and
    // every rank sees the same iteration counts for the next owner map.
    if (allgather) {  // world > 1, or a single rank exercising its exchange
      std::vector<int> owned_cnt(size_t(world), 0);
      for (const Task& t : all) owned_cnt[size_t(t.owner)] += t.w;
      const int cmax = std::max(1, *std::max_element(owned_cnt.begin(), owned_cnt.end()));
      const size_t hdr = 8 + 2 * size_t(r);
      const size_t blk = size_t(n) * size_t(cmax) + hdr;
      DBuf<double> send(dev, blk), recv(dev, blk * size_t(world));
      int col = 0;
      for (const Task& t : mine) {
        if (!fail.failed)
          MPG_CUDA(cudaMemcpyAsync(send.get() + size_t(n) * col, SOL.get() + size_t(n) * (size_t(r) * t.side + t.c0),
                                   size_t(n) * t.w * sizeof(double), cudaMemcpyDeviceToDevice, s));
        col += t.w;
      }
      std::vector<double> h(hdr, 0.0);
      h[0] = fail.failed ? 1.0 : 0.0;
      h[1] = fail.side;
      h[2] = fail.c0;
      h[3] = fail.rel;
      h[4] = fail.its;
      // plan fingerprint: every rank must have derived the same units and owners
      double fp = 0.0;
      for (const Task& t : all) fp = std::fmod(fp * 31.0 + double(t.side * 4096 + t.c0 * 16 + t.w * 4 + t.owner % 4) + 1.0, 1e15);
      h[5] = double(all.size());
      h[6] = double(cmax);
      h[7] = fp;
      for (size_t i = 0; i < mine.size(); ++i) h[8 + i] = its_mine[i];
      MPG_CUDA(cudaMemcpyAsync(send.get() + size_t(n) * size_t(cmax), h.data(), hdr * sizeof(double),
                               cudaMemcpyHostToDevice, s));
      MPG_CUDA(cudaStreamSynchronize(s));
      if (allgather(agctx, send.get(), recv.get(), int64_t(blk) * 8) != 0)
        throw CudaError("irka: allgather callback failed");
      std::vector<double> hall(hdr * size_t(world));
      for (int o = 0; o < world; ++o)
        MPG_CUDA(cudaMemcpyAsync(hall.data() + hdr * size_t(o), recv.get() + blk * size_t(o) + size_t(n) * size_t(cmax),
                                 hdr * sizeof(double), cudaMemcpyDeviceToHost, s));
      MPG_CUDA(cudaStreamSynchronize(s));
      for (int o = 0; o < world; ++o) {
        const double* ho = hall.data() + hdr * size_t(o);
        if (ho[5] != h[5] || ho[6] != h[6] || ho[7] != h[7])
          throw SolverError("irka: rank " + std::to_string(o) + " and rank " + std::to_string(rank) +
                            " derived different shard plans at sweep " + std::to_string(z) +
                            " (their reduced matrices differ)");
      }
      for (int o = 0; o < world && !fail.failed; ++o)
        if (hall[hdr * size_t(o)] != 0.0) {
          const double* ho = hall.data() + hdr * size_t(o);
          fail = Failure{true, int(ho[1]), int(ho[2]), ho[3], int(ho[4])};
        }
      std::vector<int> cursor(size_t(world), 0), ucount(size_t(world), 0);
      for (const Task& t : all) {
        const int o = t.owner;
        slot_iters[{t.side, t.c0}] = int(hall[hdr * size_t(o) + 8 + size_t(ucount[size_t(o)]++)]);
        if (!fail.failed) {
          const double* src = recv.get() + blk * size_t(o) + size_t(n) * size_t(cursor[size_t(o)]);
          MPG_CUDA(cudaMemcpyAsync(SOL.get() + size_t(n) * (size_t(r) * t.side + t.c0), src,
                                   size_t(n) * t.w * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
        cursor[size_t(o)] += t.w;
      }
      MPG_CUDA(cudaStreamSynchronize(s));
    } else {
      for (size_t i = 0; i < mine.size(); ++i) slot_iters[{mine[i].side, mine[i].c0}] = its_mine[i];
    }
    if (fail.failed) {
      char rel[32];
      std::snprintf(rel, sizeof rel, "%.3e", fail.rel);
      throw SolverError(std::string("birka: gmres did not converge on the ") + (fail.side == 0 ? "trial" : "test") +
                        " side (sweep " + std::to_string(z) + ", unit at column " + std::to_string(fail.c0) +
                        "; relative residual " + rel + " after " + std::to_string(fail.its) + " iterations)");
    }
    MPG_CUDA(cudaMemcpyAsync(X.get(), SOL.get(), size_t(n) * r * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MPG_CUDA(cudaMemcpyAsync(Y.get(), SOL.get() + size_t(n) * r, size_t(n) * r * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    orthonormalize(dev, X.get(), n, r);
    orthonormalize(dev, Y.get(), n, r);
    // ---- projection (K5) ----
    for (int j = 0; j < r; ++j) {
      launch_spmv(*op.a, X.get() + size_t(n) * j, AV.get() + size_t(n) * j, 1.0, s);
      if (op.e) launch_spmv(*op.e, X.get() + size_t(n) * j, EV.get() + size_t(n) * j, 1.0, s);
    }
    const double* ev = op.e ? EV.get() : X.get();
    const Mat er = ts_gram(dev, Y.get(), n, r, ev, n, r, n);
    const Mat ar = ts_gram(dev, Y.get(), n, r, AV.get(), n, r, n);
    host::LU lu(er);
    if (!lu.invertible())
      throw SolverError("birka: projection matrix (test basis^T trial basis) is singular at sweep " + std::to_string(z));
    kr = lu.solve(ar);
    fr = lu.solve(ts_gram(dev, Y.get(), n, r, B.get(), n, m, n));
    cr = ts_gram(dev, X.get(), n, r, C.get(), n, q, n);
    if (allgather && world > 1) {
      // Every rank projects redundantly; the ranks then adopt rank 0's reduced
      // matrices bit for bit, so the next sweep's units, owner map and stop
      // decision are identical everywhere whatever the ranks' rounding.
      const size_t cnt = size_t(r) * size_t(r + m + q);
      DBuf<double> sendr(dev, cnt), recvr(dev, cnt * size_t(world));
      std::vector<double> pack;
      pack.insert(pack.end(), kr.a.begin(), kr.a.end());
      pack.insert(pack.end(), fr.a.begin(), fr.a.end());
      pack.insert(pack.end(), cr.a.begin(), cr.a.end());
      MPG_CUDA(cudaMemcpyAsync(sendr.get(), pack.data(), cnt * 8, cudaMemcpyHostToDevice, s));
      MPG_CUDA(cudaStreamSynchronize(s));
      if (allgather(agctx, sendr.get(), recvr.get(), int64_t(cnt) * 8) != 0)
        throw CudaError("irka: allgather callback failed");
      MPG_CUDA(cudaMemcpyAsync(pack.data(), recvr.get(), cnt * 8, cudaMemcpyDeviceToHost, s));
      MPG_CUDA(cudaStreamSynchronize(s));
      std::copy(pack.begin(), pack.begin() + long(kr.a.size()), kr.a.begin());
      std::copy(pack.begin() + long(kr.a.size()), pack.begin() + long(kr.a.size() + fr.a.size()), fr.a.begin());
      std::copy(pack.begin() + long(kr.a.size() + fr.a.size()), pack.end(), cr.a.begin());
    }
    res.er = er;
    res.ar = ar;
    sweeps_done = z;
    const std::vector<host::Eig> lambda_new = host::sorted_eigenvalues(kr);
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < lambda_new.size(); ++i) {
      const double dr = lambda_new[i].re - lambda_prev[i].re, di = lambda_new[i].im - lambda_prev[i].im;
      num += dr * dr + di * di;
      den += lambda_prev[i].re * lambda_prev[i].re + lambda_prev[i].im * lambda_prev[i].im;
    }
    if (std::sqrt(num) / std::max(std::sqrt(den), 1e-300) < cfg.tol) converged = true;
    lambda_prev = lambda_new;
    if (timing)
      std::fprintf(stderr, "irka sweep %d: %.3f s (setup+builds %.3f, gmres %.3f, rest %.3f), max its %d\n", z,
                   wall() - tz0, t_build, t_gmres, wall() - tz0 - t_build - t_gmres, sweep_max_its);
    if (timing)
      for (size_t i = 0; i < lambda_new.size(); ++i)
        std::fprintf(stderr, "irka sweep %d lambda %zu %.17g %.17g\n", z, i, lambda_new[i].re, lambda_new[i].im);
  }
  res.kr = kr;
  res.fr = fr;
  res.cr = cr;
  res.lambda = lambda_prev;
  res.sweeps = sweeps_done;
  res.converged = converged;
  if (cfg.want_vw) {
    res.v.resize(size_t(n) * r);
    res.w.resize(size_t(n) * r);
    MPG_CUDA(cudaMemcpyAsync(res.v.data(), X.get(), res.v.size() * 8, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaMemcpyAsync(res.w.data(), Y.get(), res.w.size() * 8, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
  }
  return res;
}

SweepOutcome sweep_run(const ShiftedOp& op, const double* b_any, const std::vector<double>& points,
                       const SpaiOptions& spai, const GmresOptions& gmres, int mode, int max_chain_len, double* x_out) {
  if (points.empty()) throw ConfigError("spai-bench: at least one point is required");
  for (double p : points)
    if (!(p > 0.0) || !std::isfinite(p)) throw ConfigError("spai-bench: points must be positive and finite");
  if (max_chain_len < 1) throw ConfigError("spai-bench: max_chain_len must be at least 1");
  const int dev = op.device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = op.n;
  DBuf<double> b(dev, size_t(n));
  copy_in(b.get(), b_any, size_t(n), s);
  if (device_norm2(dev, b.get(), n, s) == 0.0) throw ConfigError("spai-bench: the first input column must be nonzero");
  SweepOutcome out;
  std::vector<ChainPtr> chains(points.size());
  ChainPtr chain;
  CsrPtr prev;
  // preconditioners along the sweep (bench.cpp:189-216)
  for (size_t i = 0; i < points.size(); ++i) {
    mpg_report_row row{};
    row.sweep = 1;
    row.point = int(i) + 1;
    row.kind = MPG_KIND_NONE;
    row.min_residual = row.matrix_change = row.standard_residual = std::nan("");
    if (mode != MPG_PRECOND_NONE) {
      CsrPtr a = op_explicit(op, points[i], 0.0, false);
      if (mode == MPG_PRECOND_FRESH || (mode == MPG_PRECOND_REUSE_CHAIN && (i == 0 || chain->length() + 1 > max_chain_len)) ||
          (mode == MPG_PRECOND_REUSE_FROZEN && i == 0)) {
        SpaiOutcome so = spai_or_update(a, nullptr, spai, false);
        auto ch = std::make_shared<Chain>();
        ch->factors.push_back(so.p);
        chain = ch;
        row.kind = MPG_KIND_FRESH;
        row.build_seconds = so.build_seconds;
      } else if (mode == MPG_PRECOND_REUSE_CHAIN) {
        SpaiOutcome so = spai_or_update(a, prev, spai, false);
        auto ch = std::make_shared<Chain>(*chain);
        ch->factors.push_back(so.p);
        chain = ch;
        row.kind = MPG_KIND_HORIZONTAL;
        row.build_seconds = so.build_seconds;
        row.min_residual = so.min_residual;
        row.matrix_change = so.matrix_change;
      } else {
        row.kind = MPG_KIND_REUSED_SAME_MATRIX;
      }
      prev = a;
      chains[i] = chain;
      if (n <= 5000) row.standard_residual = std_residual(a, chain);
    }
    out.rows.push_back(row);
  }
  // solves: independent once the chains exist, batched by memory
  std::vector<SolveSpec> specs(points.size());
  DBuf<double> xs(dev, x_out ? size_t(n) * points.size() : 0);
  for (size_t i = 0; i < points.size(); ++i) {
    specs[i].sre = points[i];
    specs[i].chain = chains[i];
    specs[i].b = b.get();
    specs[i].x = x_out ? xs.get() + size_t(n) * i : nullptr;
  }
  size_t free_b = 0, total_b = 0;
  MPG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double per_solve = 8.0 * double(n + 64) * double(gmres.max_iter + 8) + 1e7;
  const int per_batch = std::max(1, std::min<int>(32, int(0.7 * double(free_b) / per_solve)));
  for (size_t b0 = 0; b0 < specs.size(); b0 += size_t(per_batch)) {
    std::vector<SolveSpec> batch(specs.begin() + long(b0), specs.begin() + long(std::min(specs.size(), b0 + per_batch)));
    std::vector<GmresOutcome> oc = gmres_batch(op, batch, gmres);
    for (size_t i = 0; i < oc.size(); ++i) {
      mpg_report_row& row = out.rows[b0 + i];
      row.solves = 1;
      row.iterations = oc[i].iterations;
      row.gmres_seconds = oc[i].solve_seconds;
      out.total_iterations += oc[i].iterations;
      if (!oc[i].converged) ++out.failed;
    }
  }
  if (x_out) {
    copy_out(x_out, xs.get(), size_t(n) * points.size(), s);
    MPG_CUDA(cudaStreamSynchronize(s));
  }
  return out;
}

// ---- QB-IHOMM (proj/src/qbihomm.cpp:57-238) ----------------------------------
// Both sides' preconditioners are built first (the horizontal chain across
// points depends only on the matrices, chain.cpp:16-98); the moment solves are
// then advanced moment by moment, every (side, point) of one moment in one
// GMRES batch (solves of a moment are independent; moment j + 1 needs moment
// j's solution for its right-hand side D x_j / D^T y_j). The union basis is
// built by two-pass modified Gram-Schmidt with the reference's deflation rule
// (orth.cpp:16-40) on the device; the reduced matrices are tall-skinny Gram
// products (K5) and the quadratic term is compressed without U (x) U.
namespace {

__global__ void k_axpy(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void k_scal(double* __restrict__ y, double a, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] *= a;
}

// kron_compress_quadratic (qbihomm.cpp:210-236): thread (q, s) of a
// block owns column q r + s of the r x r^2 result and accumulates, over its
// block's rows a, out(p, t) += U(a, p) * sum_e h_e U(b_e, q) U(c_e, s).
// part[blk][p + r t]; rows with more than QC_E entries are taken in slices.
constexpr int QC_E = 8;
template <int RM>
__global__ void __launch_bounds__(RM * RM) k_qcompress(const int* __restrict__ rowptr, const int* __restrict__ bcol,
                                                       const int* __restrict__ ccol, const double* __restrict__ val,
                                                       const double* __restrict__ U, int64_t n, int r,
                                                       double* __restrict__ part) {
  __shared__ double ua[RM], ub[QC_E][RM], uc[QC_E][RM];
  __shared__ double hv[QC_E];
  const int t = threadIdx.x, q = t / RM, s = t % RM;  // blockDim = RM * RM
  const bool mine = q < r && s < r;
  double racc[RM];
#pragma unroll
  for (int p = 0; p < RM; ++p) racc[p] = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t a0 = per * blockIdx.x, a1 = min(n, a0 + per);
  for (int64_t a = a0; a < a1; ++a) {
    const int e0 = rowptr[a], e1 = rowptr[a + 1];
    if (e0 == e1) continue;
    double hsum = 0.0;
    for (int eb = e0; eb < e1; eb += QC_E) {
      const int ne = min(QC_E, e1 - eb);
      __syncthreads();
      if (t < ne * RM) {
        const int e = t / RM, j = t % RM;
        if (j < r) {
          ub[e][j] = U[bcol[eb + e] + n * j];
          uc[e][j] = U[ccol[eb + e] + n * j];
        }
        if (j == 0) hv[e] = val[eb + e];
      }
      if (eb == e0 && t < r) ua[t] = U[a + n * t];
      __syncthreads();
      if (mine)
        for (int e = 0; e < ne; ++e) hsum = fma(hv[e] * ub[e][q], uc[e][s], hsum);
    }
    if (mine) {
#pragma unroll
      for (int p = 0; p < RM; ++p)
        if (p < r) racc[p] = fma(ua[p], hsum, racc[p]);
    }
  }
  if (!mine) return;
  const int col = q * r + s;
  double* dst = part + size_t(blockIdx.x) * size_t(r) * size_t(r) * size_t(r);
#pragma unroll
  for (int p = 0; p < RM; ++p)
    if (p < r) dst[p + size_t(r) * col] = racc[p];
}

__global__ void k_sum_blocks(const double* __restrict__ part, int blocks, int64_t len, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < blocks; ++b) v += part[size_t(b) * size_t(len) + size_t(i)];
    out[i] = v;
  }
}

std::string shortest(double v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

}  // namespace

QbOutcome qbihomm_run(const ShiftedOp& op, const DevCsr& n_op, const QbH& h, const double* f_any, const double* c_any,
                      const QbSettings& cfg) {
  const int dev = op.device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = op.n;
  // QbSystem::create (qbihomm.cpp:17-43)
  if (!op.e) {
    // E = I is allowed (D = I); nothing to check
  }
  if (n_op.nrows != n || n_op.ncols != n) throw ConfigError("quadratic-bilinear system: N must be n x n");
  if (h.n != n) throw ConfigError("quadratic-bilinear system: H must be n x n^2");
  // qbihomm_reduce validation (qbihomm.cpp:146-157)
  if (cfg.sigmas.empty()) throw ConfigError("qbihomm: at least one interpolation point is required");
  for (double sg : cfg.sigmas)
    if (sg == 0.0 || !std::isfinite(sg)) throw ConfigError("qbihomm: interpolation points must be nonzero and finite");
  for (size_t i = 0; i < cfg.sigmas.size(); ++i)
    for (size_t j = i + 1; j < cfg.sigmas.size(); ++j)
      if (cfg.sigmas[i] == cfg.sigmas[j]) throw ConfigError("qbihomm: interpolation points must be distinct");
  if (cfg.p_moments < 0 || cfg.q_moments < 0) throw ConfigError("qbihomm: moment depths must be nonnegative");
  if (cfg.max_chain_len < 1) throw ConfigError("qbihomm: max_chain_len must be at least 1");

  const int ell = int(cfg.sigmas.size());
  const int depth[2] = {cfg.p_moments + cfg.q_moments, cfg.q_moments};
  const int ncols = ell * (depth[0] + 1) + ell * (depth[1] + 1);
  if (ncols > 32) throw ConfigError("qbihomm: at most 32 moment columns on the GPU path");
  DBuf<double> F(dev, size_t(n)), Cv(dev, size_t(n));
  copy_in(F.get(), f_any, size_t(n), s);
  copy_in(Cv.get(), c_any, size_t(n), s);

  // ---- preconditioners, per side along the points (qbihomm.cpp:75-108) ----
  QbOutcome out;
  std::vector<ChainPtr> chains[2];
  std::vector<mpg_report_row> build_rows[2], moment_rows[2];
  for (int side = 0; side < 2; ++side) {
    ChainPtr chain;
    CsrPtr prev;
    for (int i = 0; i < ell; ++i) {
      mpg_report_row row{};
      row.sweep = side + 1;
      row.point = i + 1;
      row.kind = MPG_KIND_NONE;
      row.min_residual = row.matrix_change = row.standard_residual = std::nan("");
      mpg_report_row mrow = row;
      mrow.kind = MPG_KIND_REUSED_SAME_MATRIX;
      const double sg = side == 0 ? cfg.sigmas[size_t(i)] : 2.0 * cfg.sigmas[size_t(i)];
      if (cfg.mode != MPG_PRECOND_NONE) {
        CsrPtr M = op_explicit(op, sg, 0.0, side == 1);
        if (cfg.mode == MPG_PRECOND_FRESH || cfg.mode == MPG_PRECOND_REUSE_FROZEN || i == 0 ||
            chain->length() + 1 > cfg.max_chain_len) {
          SpaiOutcome so = spai_or_update(M, nullptr, cfg.spai, false);
          auto ch = std::make_shared<Chain>();
          ch->factors.push_back(so.p);
          chain = ch;
          row.kind = MPG_KIND_FRESH;
          row.build_seconds = so.build_seconds;
        } else {
          SpaiOutcome so = spai_or_update(M, prev, cfg.spai, false);
          auto ch = std::make_shared<Chain>(*chain);
          ch->factors.push_back(so.p);
          chain = ch;
          row.kind = MPG_KIND_HORIZONTAL;
          row.build_seconds = so.build_seconds;
          row.min_residual = so.min_residual;
          row.matrix_change = so.matrix_change;
        }
        prev = M;
        if (n <= cfg.standard_residual_max_dim) row.standard_residual = std_residual(M, chain);
      }
      chains[side].push_back(chain);
      build_rows[side].push_back(row);
      moment_rows[side].push_back(mrow);
    }
  }

  // ---- moment solves (qbihomm.cpp:115-137) ----
  // column index of (side, point, moment) in X, in the reference's order
  auto cidx = [&](int side, int i, int j) { return side == 0 ? i * (depth[0] + 1) + j : ell * (depth[0] + 1) + i * (depth[1] + 1) + j; };
  DBuf<double> X(dev, size_t(n) * size_t(ncols)), RHS(dev, size_t(n) * size_t(2 * ell));
  const int maxd = std::max(depth[0], depth[1]);
  for (int j = 0; j <= maxd; ++j) {
    struct Job { int side, i; };
    std::vector<Job> jobs;
    std::vector<SolveSpec> specs;
    for (int side = 0; side < 2; ++side)
      for (int i = 0; i < ell; ++i) {
        if (j > depth[side]) continue;
        double* x = X.get() + size_t(n) * size_t(cidx(side, i, j));
        const double* rhs = side == 0 ? F.get() : Cv.get();
        if (j > 0) {
          double* r = RHS.get() + size_t(n) * size_t(side * ell + i);
          launch_op(op, side == 1, 1.0, 0.0, 0.0, X.get() + size_t(n) * size_t(cidx(side, i, j - 1)), r, nullptr, 1.0, s,
                    nullptr);  // D x_prev (trial) / D^T y_prev (test)
          count_launch();
          rhs = r;
        }
        if (device_norm2(dev, rhs, n, s) == 0.0) {
          MPG_CUDA(cudaMemsetAsync(x, 0, size_t(n) * sizeof(double), s));
          continue;
        }
        SolveSpec sp;
        sp.sre = side == 0 ? cfg.sigmas[size_t(i)] : 2.0 * cfg.sigmas[size_t(i)];
        sp.transpose = side == 1;
        sp.chain = chains[side][size_t(i)];
        sp.b = rhs;
        sp.x = x;
        specs.push_back(sp);
        jobs.push_back({side, i});
      }
    if (specs.empty()) continue;
    size_t free_b = 0, total_b = 0;
    MPG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double per_solve = 8.0 * double(n + 64) * double(cfg.gmres.max_iter + 8) + 1e7;
    const int per_batch = std::max(1, std::min<int>(16, int(0.7 * double(free_b) / per_solve)));
    std::vector<GmresOutcome> oc;
    for (size_t b0 = 0; b0 < specs.size(); b0 += size_t(per_batch)) {
      std::vector<SolveSpec> batch(specs.begin() + long(b0), specs.begin() + long(std::min(specs.size(), b0 + per_batch)));
      std::vector<GmresOutcome> o = gmres_batch(op, batch, cfg.gmres);
      oc.insert(oc.end(), o.begin(), o.end());
    }
    for (size_t t = 0; t < jobs.size(); ++t) {
      const Job jb = jobs[t];
      mpg_report_row& row = j == 0 ? build_rows[jb.side][size_t(jb.i)] : moment_rows[jb.side][size_t(jb.i)];
      row.solves += 1;
      row.iterations += oc[t].iterations;
      row.gmres_seconds += oc[t].solve_seconds;
      out.total_iterations += oc[t].iterations;
      out.total_solves += 1;
    }
    for (size_t t = 0; t < jobs.size(); ++t)
      if (!oc[t].converged)
        throw SolverError(std::string("qbihomm: gmres did not converge on the ") + (jobs[t].side == 0 ? "trial" : "test") +
                          " side (sigma_" + std::to_string(jobs[t].i + 1) + " = " +
                          shortest(cfg.sigmas[size_t(jobs[t].i)]) + ", moment " + std::to_string(j) +
                          "; the shifted matrix may be singular; relative residual " +
                          shortest(oc[t].final_residual / std::max(oc[t].rhs_norm, 1e-300)) + ")");
  }
  for (int side = 0; side < 2; ++side)
    for (int i = 0; i < ell; ++i) {
      out.rows.push_back(build_rows[side][size_t(i)]);
      if (moment_rows[side][size_t(i)].solves > 0) out.rows.push_back(moment_rows[side][size_t(i)]);
    }

  // ---- union basis: OrthBasis::append_block per column (orth.cpp:16-40) ----
  DBuf<double> U(dev, size_t(n) * size_t(ncols));
  const unsigned gblk = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(cx.sm_count) * 8));
  int r = 0;
  for (int col = 0; col < ncols; ++col) {
    const double* src = X.get() + size_t(n) * size_t(col);
    const double scale = std::sqrt(device_norm2(dev, src, n, s));
    if (scale == 0.0) continue;
    double* w = U.get() + size_t(n) * size_t(r);
    MPG_CUDA(cudaMemcpyAsync(w, src, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    for (int pass = 0; pass < 2; ++pass)
      for (int jj = 0; jj < r; ++jj) {
        const double* uj = U.get() + size_t(n) * size_t(jj);
        const double d = ts_gram(dev, uj, n, 1, w, n, 1, n).a[0];
        k_axpy<<<gblk, 256, 0, s>>>(w, -d, uj, n);
        MPG_CHECK_LAUNCH();
        count_launch();
      }
    const double nrm = std::sqrt(device_norm2(dev, w, n, s));
    if (nrm <= 1e-10 * scale) continue;
    k_scal<<<gblk, 256, 0, s>>>(w, 1.0 / nrm, n);
    MPG_CHECK_LAUNCH();
    count_launch();
    ++r;
  }
  if (r == 0) throw SolverError("qbihomm: the collected moment columns are all zero");
  out.r = r;

  // ---- projections (qbihomm.cpp:195-203) ----
  DBuf<double> T(dev, size_t(n) * size_t(r));
  for (int which = 0; which < 3; ++which) {
    for (int jj = 0; jj < r; ++jj) {
      const double* uj = U.get() + size_t(n) * size_t(jj);
      double* tj = T.get() + size_t(n) * size_t(jj);
      if (which == 0) launch_op(op, false, 1.0, 0.0, 0.0, uj, tj, nullptr, 1.0, s, nullptr);  // D u
      else launch_spmv(which == 1 ? *op.a : n_op, uj, tj, 1.0, s);                             // K u, N u
      count_launch();
    }
    (which == 0 ? out.d : which == 1 ? out.k : out.n_op) = ts_gram(dev, U.get(), n, r, T.get(), n, r, n);
  }
  out.f = ts_gram(dev, U.get(), n, r, F.get(), n, 1, n);
  out.c = ts_gram(dev, U.get(), n, r, Cv.get(), n, 1, n);
  {
    const int blocks = int(std::min<int64_t>(int64_t(cx.sm_count) * 2, std::max<int64_t>(1, n)));
    const int64_t len = int64_t(r) * r * r;
    DBuf<double> part(dev, size_t(blocks) * size_t(len)), hred(dev, size_t(len));
    if (r <= 8)
      k_qcompress<8><<<blocks, 64, 0, s>>>(h.rowptr.get(), h.bcol.get(), h.ccol.get(), h.val.get(), U.get(), n, r,
                                           part.get());
    else if (r <= 16)
      k_qcompress<16><<<blocks, 256, 0, s>>>(h.rowptr.get(), h.bcol.get(), h.ccol.get(), h.val.get(), U.get(), n, r,
                                             part.get());
    else
      k_qcompress<32><<<blocks, 1024, 0, s>>>(h.rowptr.get(), h.bcol.get(), h.ccol.get(), h.val.get(), U.get(), n, r,
                                              part.get());
    MPG_CHECK_LAUNCH();
    k_sum_blocks<<<unsigned((len + 255) / 256), 256, 0, s>>>(part.get(), blocks, len, hred.get());
    MPG_CHECK_LAUNCH();
    count_launch(2);
    out.h = Mat(r, r * r);
    MPG_CUDA(cudaMemcpyAsync(out.h.a.data(), hred.get(), size_t(len) * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  out.basis = DBuf<double>(dev, size_t(n) * size_t(r));
  MPG_CUDA(cudaMemcpyAsync(out.basis.get(), U.get(), size_t(n) * size_t(r) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  return out;
}

// ---- second-order transfer-function error (proj/src/airga.cpp:80-85, :386-447) -----
namespace {
__global__ void k_comb3(const double* __restrict__ vm, const double* __restrict__ vd, const double* __restrict__ vk,
                        double a, double b, int64_t nnz, double* __restrict__ out, unsigned long long* zeros) {
  unsigned long long z = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = a * vm[i] + b * vd[i] + vk[i];
    out[i] = v;
    z += v == 0.0;
  }
  if (z) atomicAdd(zeros, z);
}
__global__ void k_comb3w(const double* __restrict__ vm, const double* __restrict__ vd, const double* __restrict__ vk,
                         double a, double b, double c, int64_t nnz, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = a * vm[i] + b * vd[i] + c * vk[i];
}
}  // namespace


namespace {
// s^2 M + s D + K on the merged pattern of M, D, K (aligned, zero-filled value
// arrays built once); at(s) forms one matrix with one kernel and drops exact
// zeros as linear_combination does (sparse.cpp:191, airga.cpp:80-85).
struct Pencil3 {
  int dev = 0;
  int64_t n = 0, unnz = 0;
  std::vector<int> urp, uci;
  DBuf<int> drp, dci;
  DBuf<double> dv[3];
  Pencil3(const CsrPtr& m, const CsrPtr& d, const CsrPtr& k) : dev(m->device), n(m->nrows) {
    cudaStream_t s = ctx(dev).stream;
    std::vector<int> rp3[3], ci3[3];
    std::vector<double> v3[3];
    const CsrPtr src[3] = {m, d, k};
    for (int t = 0; t < 3; ++t) {
      const DevCsr& a = *src[t];
      rp3[t].resize(size_t(n) + 1);
      ci3[t].resize(size_t(a.nnz));
      v3[t].resize(size_t(a.nnz));
      MPG_CUDA(cudaMemcpyAsync(rp3[t].data(), a.rowptr.get(), rp3[t].size() * 4, cudaMemcpyDeviceToHost, s));
      if (a.nnz) {
        MPG_CUDA(cudaMemcpyAsync(ci3[t].data(), a.colind.get(), ci3[t].size() * 4, cudaMemcpyDeviceToHost, s));
        MPG_CUDA(cudaMemcpyAsync(v3[t].data(), a.val.get(), v3[t].size() * 8, cudaMemcpyDeviceToHost, s));
      }
    }
    MPG_CUDA(cudaStreamSynchronize(s));
    urp.assign(size_t(n) + 1, 0);
    std::vector<double> uv[3];
    for (int64_t i = 0; i < n; ++i) {
      int p[3] = {rp3[0][size_t(i)], rp3[1][size_t(i)], rp3[2][size_t(i)]};
      while (true) {
        int c = INT32_MAX;
        for (int t = 0; t < 3; ++t)
          if (p[t] < rp3[t][size_t(i) + 1]) c = std::min(c, ci3[t][size_t(p[t])]);
        if (c == INT32_MAX) break;
        uci.push_back(c);
        for (int t = 0; t < 3; ++t) {
          double v = 0.0;
          while (p[t] < rp3[t][size_t(i) + 1] && ci3[t][size_t(p[t])] == c) v += v3[t][size_t(p[t]++)];
          uv[t].push_back(v);
        }
      }
      urp[size_t(i) + 1] = int(uci.size());
    }
    unnz = int64_t(uci.size());
    drp = DBuf<int>(dev, urp.size());
    dci = DBuf<int>(dev, std::max<size_t>(1, uci.size()));
    MPG_CUDA(cudaMemcpyAsync(drp.get(), urp.data(), urp.size() * 4, cudaMemcpyHostToDevice, s));
    if (unnz) MPG_CUDA(cudaMemcpyAsync(dci.get(), uci.data(), uci.size() * 4, cudaMemcpyHostToDevice, s));
    for (int t = 0; t < 3; ++t) {
      dv[t] = DBuf<double>(dev, std::max<size_t>(1, uv[t].size()));
      if (unnz) MPG_CUDA(cudaMemcpyAsync(dv[t].get(), uv[t].data(), uv[t].size() * 8, cudaMemcpyHostToDevice, s));
    }
    MPG_CUDA(cudaStreamSynchronize(s));
  }
  // ||cm M + cd D + ck K||_F
  double combo_norm(double cm, double cd, double ck) const {
    auto& cx = ctx(dev);
    cudaStream_t s = cx.stream;
    if (unnz == 0) return 0.0;
    DBuf<double> vals(dev, size_t(unnz));
    k_comb3w<<<unsigned(std::min<int64_t>((unnz + 255) / 256, int64_t(cx.sm_count) * 8)), 256, 0, s>>>(
        dv[0].get(), dv[1].get(), dv[2].get(), cm, cd, ck, unnz, vals.get());
    MPG_CHECK_LAUNCH();
    count_launch();
    return std::sqrt(device_norm2(dev, vals.get(), unnz, s));
  }
  CsrPtr at(double sv) const {
    auto& cx = ctx(dev);
    cudaStream_t s = cx.stream;
    DBuf<double> vals(dev, std::max<size_t>(1, size_t(unnz)));
    DBuf<unsigned long long> zeros(dev, 1);
    MPG_CUDA(cudaMemsetAsync(zeros.get(), 0, sizeof(unsigned long long), s));
    if (unnz) {
      k_comb3<<<unsigned(std::min<int64_t>((unnz + 255) / 256, int64_t(cx.sm_count) * 8)), 256, 0, s>>>(
          dv[0].get(), dv[1].get(), dv[2].get(), sv * sv, sv, unnz, vals.get(), zeros.get());
      MPG_CHECK_LAUNCH();
      count_launch();
    }
    unsigned long long nz0 = 0;
    MPG_CUDA(cudaMemcpyAsync(&nz0, zeros.get(), sizeof nz0, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
    if (nz0 == 0) {
      DBuf<int> rp2(dev, urp.size()), ci2(dev, std::max<size_t>(1, uci.size()));
      MPG_CUDA(cudaMemcpyAsync(rp2.get(), drp.get(), urp.size() * 4, cudaMemcpyDeviceToDevice, s));
      if (unnz) MPG_CUDA(cudaMemcpyAsync(ci2.get(), dci.get(), uci.size() * 4, cudaMemcpyDeviceToDevice, s));
      return csr_from_device_parts(dev, n, n, std::move(rp2), std::move(ci2), std::move(vals));
    }
    std::vector<double> hv(static_cast<size_t>(unnz));
    MPG_CUDA(cudaMemcpyAsync(hv.data(), vals.get(), hv.size() * 8, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> rp64(size_t(n) + 1, 0), ci64;
    std::vector<double> v64;
    for (int64_t i = 0; i < n; ++i) {
      for (int q = urp[size_t(i)]; q < urp[size_t(i) + 1]; ++q)
        if (hv[size_t(q)] != 0.0) {
          ci64.push_back(uci[size_t(q)]);
          v64.push_back(hv[size_t(q)]);
        }
      rp64[size_t(i) + 1] = int64_t(ci64.size());
    }
    return csr_from_host(dev, n, n, rp64.data(), ci64.data(), v64.data());
  }
};
}  // namespace

std::vector<double> tf_error_run(const CsrPtr& m, const CsrPtr& d, const CsrPtr& k, const double* f_any, int n_in,
                                 const double* c_any, int n_out, const host::Mat& rm, const host::Mat& rd,
                                 const host::Mat& rk, const host::Mat& rf, const host::Mat& rc,
                                 const std::vector<double>& grid, const TfSettings& cfg, long long* total_iterations) {
  const int dev = m->device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = m->nrows;
  for (const CsrPtr& x : {m, d, k})
    if (x->nrows != n || x->ncols != n || x->device != dev)
      throw std::invalid_argument("transfer_function_error: M, D, K must be n x n on one device");
  const int r = rm.rows;
  if (rm.cols != r || rd.rows != r || rd.cols != r || rk.rows != r || rk.cols != r || rf.rows != r ||
      rf.cols != n_in || rc.rows != r || rc.cols != n_out)
    throw std::invalid_argument("transfer_function_error: reduced model shapes do not match");
  if (n_in < 1 || n_out < 1 || n_out * n_in > 1024) throw std::invalid_argument("transfer_function_error: bad F / C");
  const Pencil3 pencil(m, d, k);
  DBuf<double> F(dev, size_t(n) * n_in), Cm(dev, size_t(n) * n_out), X(dev, size_t(n) * n_in);
  copy_in(F.get(), f_any, size_t(n) * n_in, s);
  copy_in(Cm.get(), c_any, size_t(n) * n_out, s);
  std::vector<double> fnorm(static_cast<size_t>(n_in));
  for (int j = 0; j < n_in; ++j) fnorm[size_t(j)] = device_norm2(dev, F.get() + size_t(n) * j, n, s);

  std::vector<double> errors(grid.size(), std::numeric_limits<double>::quiet_NaN());
  ChainPtr chain;
  CsrPtr chain_matrix;
  long long its = 0;
  for (size_t g = 0; g < grid.size(); ++g) {
    const double sv = grid[g];
    if (!(sv > 0.0) || !std::isfinite(sv)) continue;
    const CsrPtr A = pencil.at(sv);
    ChainPtr prec;
    if (cfg.mode == MPG_PRECOND_FRESH) {
      auto ch = std::make_shared<Chain>();
      ch->factors.push_back(spai_or_update(A, nullptr, cfg.spai, false).p);
      prec = ch;
    } else if (cfg.mode == MPG_PRECOND_REUSE_CHAIN || cfg.mode == MPG_PRECOND_REUSE_FROZEN) {
      if (!chain || chain->length() + 1 > cfg.max_chain_len) {
        auto ch = std::make_shared<Chain>();
        ch->factors.push_back(spai_or_update(A, nullptr, cfg.spai, false).p);
        chain = ch;
      } else if (cfg.mode == MPG_PRECOND_REUSE_CHAIN) {
        auto ch = std::make_shared<Chain>(*chain);
        ch->factors.push_back(spai_or_update(A, chain_matrix, cfg.spai, false).p);
        chain = ch;
      }
      chain_matrix = A;
      prec = chain;
    }
    OpPtr op = op_create(A, nullptr);
    std::vector<SolveSpec> specs;
    std::vector<int> cols;
    for (int j = 0; j < n_in; ++j) {
      double* xj = X.get() + size_t(n) * j;
      if (fnorm[size_t(j)] == 0.0) {
        MPG_CUDA(cudaMemsetAsync(xj, 0, size_t(n) * sizeof(double), s));
        continue;
      }
      SolveSpec sp;
      sp.sre = 0.0;
      sp.ca = 1.0;  // y = A(s) x
      sp.chain = prec;
      sp.b = F.get() + size_t(n) * j;
      sp.x = xj;
      specs.push_back(sp);
      cols.push_back(j);
    }
    bool ok = true;
    if (!specs.empty()) {
      const std::vector<GmresOutcome> oc = gmres_batch(*op, specs, cfg.gmres);
      for (const auto& o : oc) {
        ok = ok && o.converged;
        its += o.iterations;
      }
    }
    if (!ok) continue;
    const Mat h = ts_gram(dev, Cm.get(), n, n_out, X.get(), n, n_in, n);  // C^T X
    Mat ar(r, r);
    for (size_t i = 0; i < ar.a.size(); ++i) ar.a[i] = sv * sv * rm.a[i] + sv * rd.a[i] + rk.a[i];
    const host::LU lu(ar);
    if (!lu.invertible()) continue;
    const Mat hr = host::mul(host::transpose(rc), lu.solve(rf));
    const double denom = host::fro(h);
    if (denom == 0.0) continue;
    Mat diff = h;
    for (size_t i = 0; i < diff.a.size(); ++i) diff.a[i] -= hr.a[i];
    errors[g] = host::fro(diff) / denom;
  }
  if (total_iterations) *total_iterations = its;
  return errors;
}

// ---- AIRGA (proj/src/airga.cpp:136-317) --------------------------------------------
// Per sweep and expansion point: A(s_i) = s_i^2 M + s_i D + K from the merged
// pattern, the preconditioner by mode (ReuseChain: fresh at the very first
// point, horizontal updates along a sweep, a vertical update into the next
// sweep's first point), the zeroth-moment block A X = F (n_in solves in one
// batch), then higher moments A X = -M X_prev until the basis is full, nothing
// new is appended, or the inner H2 gap drops below inner_tol; the basis is
// OrthBasis (block scale = largest singular value, two-pass MGS, 1e-10
// deflation) on the device; the reduced model and H2 gaps on the host.
namespace {
std::string airga_shortest(double v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}
}  // namespace

AirgaOutcome airga_run(const CsrPtr& m, const CsrPtr& d, const CsrPtr& k, const double* f_any, int n_in,
                       const double* c_any, int n_out, const AirgaSettings& cfg) {
  const int dev = m->device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = m->nrows;
  for (const CsrPtr& x : {m, d, k})
    if (x->nrows != n || x->ncols != n || x->device != dev)
      throw ConfigError("second-order system: M, D, K must be n x n on one device");
  if (n_in < 1 || n_out < 1) throw ConfigError("second-order system: F and C need at least one column");
  std::vector<double> points = cfg.points;
  if (points.empty()) throw ConfigError("airga: at least one expansion point is required");
  std::sort(points.begin(), points.end());
  for (double sp : points)
    if (!(sp > 0.0) || !std::isfinite(sp)) throw ConfigError("airga: expansion points must be positive and finite");
  if (std::adjacent_find(points.begin(), points.end()) != points.end())
    throw ConfigError("airga: expansion points must be distinct");
  const int ell = int(points.size());
  if (cfg.r_max < ell)
    throw ConfigError("airga: r_max (" + std::to_string(cfg.r_max) + ") must be at least the number of expansion points (" +
                      std::to_string(ell) + ")");
  if (cfg.max_outer < 1) throw ConfigError("airga: max_outer must be at least 1");
  if (cfg.max_chain_len < 1) throw ConfigError("airga: max_chain_len must be at least 1");
  if (cfg.r_max > 32 || n_in * n_out > 1024) throw ConfigError("airga: r_max <= 32 on the GPU path");

  AirgaOutcome out;
  const Pencil3 pencil(m, d, k);
  {  // proportionality warning (airga.cpp:167-174)
    const double dnorm = pencil.combo_norm(0.0, 1.0, 0.0);
    const double defect = pencil.combo_norm(-cfg.alpha, 1.0, -cfg.beta);
    if (dnorm > 0.0 && defect > 1e-12 * dnorm)
      out.warnings.push_back("damping deviates from alpha*M + beta*K (relative defect " +
                             airga_shortest(defect / dnorm) + "); reduction proceeds on D as given");
  }
  DBuf<double> F(dev, size_t(n) * n_in), Cm(dev, size_t(n) * n_out);
  copy_in(F.get(), f_any, size_t(n) * n_in, s);
  copy_in(Cm.get(), c_any, size_t(n) * n_out, s);
  const int cap = cfg.r_max;
  DBuf<double> U(dev, size_t(n) * cap), T(dev, size_t(n) * cap);
  std::vector<DBuf<double>> blocks;
  for (int i = 0; i < ell; ++i) blocks.emplace_back(dev, size_t(n) * n_in);
  DBuf<double> RHS(dev, size_t(n) * n_in);
  const unsigned gblk = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(cx.sm_count) * 8));
  auto dot = [&](const double* x, const double* y) { return ts_gram(dev, x, n, 1, y, n, 1, n).a[0]; };

  ChainPtr prev_first_chain;
  CsrPtr prev_first_matrix;
  host::StateSpace prev_ss;
  bool have_prev = false;
  for (int z = 1; z <= cfg.max_outer; ++z) {
    int size = 0;
    std::vector<CsrPtr> a_ops;
    for (double sp : points) a_ops.push_back(pencil.at(sp));
    std::vector<ChainPtr> chains(static_cast<size_t>(ell));
    std::vector<OpPtr> ops;
    for (int i = 0; i < ell; ++i) ops.push_back(op_create(a_ops[size_t(i)], nullptr));
    auto solve_block = [&](int i, const double* rhs, double sign, int moment, mpg_report_row& row) {
      std::vector<SolveSpec> specs;
      std::vector<int> cols;
      double* xb = blocks[size_t(i)].get();
      for (int j = 0; j < n_in; ++j) {
        const double* bj = rhs + size_t(n) * j;
        if (device_norm2(dev, bj, n, s) == 0.0) {
          MPG_CUDA(cudaMemsetAsync(xb + size_t(n) * j, 0, size_t(n) * sizeof(double), s));
          continue;
        }
        SolveSpec sp;
        sp.sre = 0.0;
        sp.ca = 1.0;
        sp.chain = chains[size_t(i)];
        sp.b = bj;
        sp.x = xb + size_t(n) * j;
        specs.push_back(sp);
        cols.push_back(j);
      }
      if (specs.empty()) return;
      const std::vector<GmresOutcome> oc = gmres_batch(*ops[size_t(i)], specs, cfg.gmres);
      for (size_t t = 0; t < oc.size(); ++t) {
        row.solves += 1;
        row.iterations += oc[t].iterations;
        row.gmres_seconds += oc[t].solve_seconds;
        if (!oc[t].converged)
          throw SolverError("gmres did not converge (sweep " + std::to_string(z) + ", point " + std::to_string(i + 1) +
                            ", moment " + std::to_string(moment) + ", column " + std::to_string(cols[t]) +
                            "; relative residual " +
                            airga_shortest(oc[t].final_residual / std::max(oc[t].rhs_norm, 1e-300)) + " after " +
                            std::to_string(oc[t].iterations) + " iterations)");
        if (sign != 1.0) {
          k_scal<<<gblk, 256, 0, s>>>(xb + size_t(n) * cols[t], sign, n);
          MPG_CHECK_LAUNCH();
          count_launch();
        }
      }
    };
    // OrthBasis::append_block (orth.cpp:16-40); returns the columns kept
    auto append_block = [&](const double* blk) {
      const Mat g = ts_gram(dev, blk, n, n_in, blk, n, n_in, n);
      double smax = 0.0;
      if (n_in == 1) {
        smax = std::sqrt(std::max(g.a[0], 0.0));
      } else {
        for (const host::Eig& e : host::eigenvalues(g)) smax = std::max(smax, e.re);
        smax = std::sqrt(std::max(smax, 0.0));
      }
      if (smax == 0.0) return 0;
      const double cutoff = 1e-10 * smax;
      int kept = 0;
      for (int c = 0; c < n_in && size < cap; ++c) {
        double* w = U.get() + size_t(n) * size_t(size);
        MPG_CUDA(cudaMemcpyAsync(w, blk + size_t(n) * c, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
        for (int pass = 0; pass < 2; ++pass)
          for (int j = 0; j < size; ++j) {
            const double* uj = U.get() + size_t(n) * size_t(j);
            const double dd = dot(uj, w);
            k_axpy<<<gblk, 256, 0, s>>>(w, -dd, uj, n);
            MPG_CHECK_LAUNCH();
            count_launch();
          }
        const double nrm = std::sqrt(device_norm2(dev, w, n, s));
        if (nrm <= cutoff) continue;
        k_scal<<<gblk, 256, 0, s>>>(w, 1.0 / nrm, n);
        MPG_CHECK_LAUNCH();
        count_launch();
        ++size;
        ++kept;
      }
      return kept;
    };
    auto project = [&]() {
      host::Mat rm, rd, rk;
      for (int which = 0; which < 3; ++which) {
        const DevCsr& a = which == 0 ? *m : which == 1 ? *d : *k;
        for (int j = 0; j < size; ++j) {
          launch_spmv(a, U.get() + size_t(n) * j, T.get() + size_t(n) * j, 1.0, s);
          count_launch();
        }
        (which == 0 ? rm : which == 1 ? rd : rk) = ts_gram(dev, U.get(), n, size, T.get(), n, size, n);
      }
      out.m = rm;
      out.d = rd;
      out.k = rk;
      out.f = ts_gram(dev, U.get(), n, size, F.get(), n, n_in, n);
      out.c = ts_gram(dev, U.get(), n, size, Cm.get(), n, n_out, n);
      return host::second_order_to_state_space(out.m, out.d, out.k, out.f, out.c);
    };
    auto h2_gap = [](const host::StateSpace& p, const host::StateSpace& q) {
      const double dist = host::h2_distance(p, q);
      if (!std::isfinite(dist)) return std::numeric_limits<double>::infinity();
      const double scale = host::h2_norm(q);
      if (!std::isfinite(scale)) return std::numeric_limits<double>::infinity();
      return dist / std::max(1.0, scale);
    };
    // zeroth moments with the preconditioners (airga.cpp:196-262)
    for (int i = 0; i < ell; ++i) {
      mpg_report_row row{};
      row.sweep = z;
      row.point = i + 1;
      row.kind = MPG_KIND_NONE;
      row.min_residual = row.matrix_change = row.standard_residual = std::nan("");
      const CsrPtr& A = a_ops[size_t(i)];
      if (cfg.mode == MPG_PRECOND_FRESH) {
        SpaiOutcome so = spai_or_update(A, nullptr, cfg.spai, false);
        auto ch = std::make_shared<Chain>();
        ch->factors.push_back(so.p);
        chains[size_t(i)] = ch;
        row.kind = MPG_KIND_FRESH;
        row.build_seconds = so.build_seconds;
      } else if (cfg.mode == MPG_PRECOND_REUSE_CHAIN || cfg.mode == MPG_PRECOND_REUSE_FROZEN) {
        const bool first_ever = z == 1 && i == 0;
        const ChainPtr parent = i == 0 ? (z == 1 ? nullptr : prev_first_chain) : chains[size_t(i) - 1];
        if (first_ever || parent->length() + 1 > cfg.max_chain_len) {
          SpaiOutcome so = spai_or_update(A, nullptr, cfg.spai, false);
          auto ch = std::make_shared<Chain>();
          ch->factors.push_back(so.p);
          chains[size_t(i)] = ch;
          row.kind = MPG_KIND_FRESH;
          row.build_seconds = so.build_seconds;
        } else {
          const CsrPtr a_prev = i == 0 ? prev_first_matrix : a_ops[size_t(i) - 1];
          SpaiOutcome so = spai_or_update(A, a_prev, cfg.spai, false);
          auto ch = std::make_shared<Chain>(*parent);
          ch->factors.push_back(so.p);
          chains[size_t(i)] = ch;
          row.kind = i == 0 ? MPG_KIND_VERTICAL : MPG_KIND_HORIZONTAL;
          row.build_seconds = so.build_seconds;
          row.min_residual = so.min_residual;
          row.matrix_change = so.matrix_change;
        }
      }
      solve_block(i, F.get(), 1.0, 0, row);
      if (cfg.mode != MPG_PRECOND_NONE && n <= cfg.standard_residual_max_dim)
        row.standard_residual = std_residual(A, chains[size_t(i)]);
      out.rows.push_back(row);
    }
    for (int i = 0; i < ell; ++i) append_block(blocks[size_t(i)].get());
    host::StateSpace red_ss = project();
    std::vector<mpg_report_row> mrows(static_cast<size_t>(ell));
    for (int i = 0; i < ell; ++i) {
      mrows[size_t(i)] = mpg_report_row{};
      mrows[size_t(i)].sweep = z;
      mrows[size_t(i)].point = i + 1;
      mrows[size_t(i)].kind = MPG_KIND_REUSED_SAME_MATRIX;
      mrows[size_t(i)].min_residual = mrows[size_t(i)].matrix_change = mrows[size_t(i)].standard_residual = std::nan("");
    }
    for (int j = 1; size < cap; ++j) {  // higher moments (airga.cpp:272-292)
      bool appended = false;
      for (int i = 0; i < ell && size < cap; ++i) {
        for (int c = 0; c < n_in; ++c) {
          launch_spmv(*m, blocks[size_t(i)].get() + size_t(n) * c, RHS.get() + size_t(n) * c, 1.0, s);
          count_launch();
        }
        solve_block(i, RHS.get(), -1.0, j, mrows[size_t(i)]);
        if (append_block(blocks[size_t(i)].get()) > 0) appended = true;
      }
      if (!appended) break;
      host::StateSpace next_ss = project();
      const double gap = h2_gap(red_ss, next_ss);
      red_ss = next_ss;
      if (gap <= cfg.inner_tol) break;
    }
    if (size >= cap && cfg.r_max > ell)
      out.warnings.push_back("sweep " + std::to_string(z) + ": basis reached r_max before inner convergence");
    for (const auto& r : mrows)
      if (r.solves > 0) out.rows.push_back(r);
    out.sweeps = z;
    out.r = size;
    out.final_points = points;
    out.basis = DBuf<double>(dev, size_t(n) * std::max(size, 1));
    MPG_CUDA(cudaMemcpyAsync(out.basis.get(), U.get(), size_t(n) * size * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (have_prev && h2_gap(prev_ss, red_ss) <= cfg.outer_tol) {
      out.converged = true;
      break;
    }
    prev_ss = red_ss;
    have_prev = true;
    if (cfg.mode == MPG_PRECOND_REUSE_CHAIN || cfg.mode == MPG_PRECOND_REUSE_FROZEN) {
      prev_first_chain = chains[0];
      prev_first_matrix = a_ops[0];
    }
    if (z < cfg.max_outer) points = host::update_expansion_points(out.m, out.d, out.k, points);
  }
  if (!out.converged)
    out.warnings.push_back("outer loop left unconverged after " + std::to_string(out.sweeps) + " sweeps");
  MPG_CUDA(cudaStreamSynchronize(s));
  return out;
}

// ---- BIRKA with couplings (proj/src/birka.cpp:139-310, kron.cpp:34-131) ------------
namespace {
struct HostCsr32 {
  int64_t n = 0;
  std::vector<int> rp, ci;
  std::vector<double> v;
};
HostCsr32 download_csr(const DevCsr& a) {
  HostCsr32 h;
  h.n = a.nrows;
  h.rp.resize(size_t(a.nrows) + 1);
  h.ci.resize(size_t(a.nnz));
  h.v.resize(size_t(a.nnz));
  cudaStream_t s = ctx(a.device).stream;
  MPG_CUDA(cudaMemcpyAsync(h.rp.data(), a.rowptr.get(), h.rp.size() * 4, cudaMemcpyDeviceToHost, s));
  if (a.nnz) {
    MPG_CUDA(cudaMemcpyAsync(h.ci.data(), a.colind.get(), h.ci.size() * 4, cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaMemcpyAsync(h.v.data(), a.val.get(), h.v.size() * 8, cudaMemcpyDeviceToHost, s));
  }
  MPG_CUDA(cudaStreamSynchronize(s));
  return h;
}
HostCsr32 transpose_host(const HostCsr32& a) {
  HostCsr32 t;
  t.n = a.n;
  t.rp.assign(size_t(a.n) + 1, 0);
  for (int c : a.ci) ++t.rp[size_t(c) + 1];
  for (int64_t i = 0; i < a.n; ++i) t.rp[size_t(i) + 1] += t.rp[size_t(i)];
  t.ci.resize(a.ci.size());
  t.v.resize(a.v.size());
  std::vector<int> pos(t.rp.begin(), t.rp.end() - 1);
  for (int64_t i = 0; i < a.n; ++i)
    for (int k = a.rp[size_t(i)]; k < a.rp[size_t(i) + 1]; ++k) {
      const int c = a.ci[size_t(k)];
      t.ci[size_t(pos[size_t(c)])] = int(i);
      t.v[size_t(pos[size_t(c)]++)] = a.v[size_t(k)];
    }
  return t;
}
// assemble_explicit (kron.cpp:72-131): -(Lambda (x) I) - (I (x) K) - sum (S^T (x) N); the
// triplets are generated row by row, so each row is built sorted and summed directly.
CsrPtr assemble_kron(int dev, const Mat& lam, const HostCsr32& k, const std::vector<std::pair<Mat, const HostCsr32*>>& cps,
                     int64_t& estimate) {
  const int64_t n = k.n;
  const int r = lam.rows;
  int64_t lnz = 0;
  for (double x : lam.a) lnz += x != 0.0;
  estimate = lnz * n + int64_t(r) * int64_t(k.v.size());
  for (const auto& cp : cps) {
    int64_t snz = 0;
    for (double x : cp.first.a) snz += x != 0.0;
    estimate += snz * int64_t(cp.second->v.size());
  }
  std::vector<int64_t> rp(size_t(n * r) + 1, 0), ci;
  std::vector<double> vv;
  std::vector<std::pair<int64_t, double>> row;
  for (int bi = 0; bi < r; ++bi)
    for (int64_t i = 0; i < n; ++i) {
      row.clear();
      for (int bj = 0; bj < r; ++bj)
        if (lam(bi, bj) != 0.0) row.push_back({bj * n + i, -lam(bi, bj)});
      for (int kk = k.rp[size_t(i)]; kk < k.rp[size_t(i) + 1]; ++kk) row.push_back({bi * n + k.ci[size_t(kk)], -k.v[size_t(kk)]});
      for (const auto& cp : cps)
        for (int bj = 0; bj < r; ++bj) {
          const double sv = cp.first(bj, bi);
          if (sv == 0.0) continue;
          const HostCsr32& nm = *cp.second;
          for (int kk = nm.rp[size_t(i)]; kk < nm.rp[size_t(i) + 1]; ++kk)
            row.push_back({bj * n + nm.ci[size_t(kk)], -sv * nm.v[size_t(kk)]});
        }
      std::stable_sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (size_t p = 0; p < row.size();) {
        const int64_t c = row[p].first;
        double sum = 0.0;
        while (p < row.size() && row[p].first == c) sum += row[p++].second;
        ci.push_back(c);
        vv.push_back(sum);
      }
      rp[size_t(bi * n + i) + 1] = int64_t(ci.size());
    }
  return csr_from_host(dev, n * r, n * r, rp.data(), ci.data(), vv.data());
}
}  // namespace

BirkaOutcome birka_coupled_run(const CsrPtr& kp, const std::vector<CsrPtr>& n_ops, const double* b_any, int m,
                               const double* c_any, int q, const IrkaSettings& cfg, long long explicit_nnz_cap) {
  const int dev = kp->device;
  auto& cx = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = cx.stream;
  const int64_t n = kp->nrows;
  const int r = cfg.r;
  if (kp->ncols != n) throw ConfigError("bilinear system: K must be square");
  if (m < 1 || q < 1) throw ConfigError("bilinear system: F and C need at least one column");
  if (int(n_ops.size()) != m) throw ConfigError("bilinear system: one N per input is required");
  for (const auto& nj : n_ops)
    if (nj->nrows != n || nj->ncols != n || nj->device != dev) throw ConfigError("bilinear system: every N must be n x n");
  if (cfg.max_sweeps < 1) throw ConfigError("birka: max_sweeps must be at least 1");
  if (cfg.max_chain_len < 1) throw ConfigError("birka: max_chain_len must be at least 1");
  if (r < 1 || int64_t(r) > n) throw ConfigError("birka: reduced order must be in [1, n]");
  if (r > 32) throw ConfigError("birka: r <= 32 on the GPU path");

  const HostCsr32 kh = download_csr(*kp), kt = transpose_host(kh);
  std::vector<HostCsr32> nh, nt;
  for (const auto& nj : n_ops) {
    nh.push_back(download_csr(*nj));
    nt.push_back(transpose_host(nh.back()));
  }
  std::vector<double> B(size_t(n) * m), Cc(size_t(n) * q);
  copy_out(B.data(), b_any, B.size(), s);  // any memory -> host
  copy_out(Cc.data(), c_any, Cc.size(), s);
  MPG_CUDA(cudaStreamSynchronize(s));
  DBuf<double> Bd(dev, B.size()), Cd(dev, Cc.size());
  copy_in(Bd.get(), B.data(), B.size(), s);
  copy_in(Cd.get(), Cc.data(), Cc.size(), s);

  BirkaOutcome out;
  Mat kr(r, r), fr(r, m), cr(r, q);
  std::vector<Mat> nr(size_t(m), Mat(r, r));
  default_seed(*kp, cfg, kr, fr, cr, s);
  struct Side {
    ChainPtr chain;
    CsrPtr prev;
    bool degraded = false;
  } sides[2];
  std::mt19937_64 perturb_rng(cfg.seed ^ 0x9e3779b97f4a7c15ull);
  std::vector<host::Eig> lambda_prev = host::sorted_eigenvalues(kr);
  DBuf<double> X(dev, size_t(n) * r), Y(dev, size_t(n) * r), T(dev, size_t(n) * r);
  for (int z = 1; z <= cfg.max_sweeps && !out.converged; ++z) {
    host::Spectrum spec;
    if (!host::real_spectrum(kr, spec)) {
      std::uniform_real_distribution<double> unit(-1.0, 1.0);
      Mat nudged = kr;
      const double scale = 1e-8 * std::max(1.0, host::fro(kr));
      for (double& v : nudged.a) v += scale * unit(perturb_rng);
      if (!host::real_spectrum(nudged, spec))
        throw SolverError("birka: reduced state matrix is not diagonalizable (sweep " + std::to_string(z) +
                          "), even after perturbation");
      kr = nudged;
      lambda_prev = host::sorted_eigenvalues(kr);
    }
    const Mat rinv_t = host::transpose(spec.basis_inv);
    const Mat f2 = host::mul(host::transpose(fr), rinv_t);    // m x r
    const Mat c2 = host::mul(host::transpose(cr), spec.basis);  // q x r
    std::vector<std::pair<Mat, const HostCsr32*>> cps[2];
    for (int j = 0; j < m; ++j) {
      const Mat n2 = host::mul(host::mul(host::transpose(spec.basis), nr[size_t(j)]), rinv_t);
      cps[0].push_back({n2, &nh[size_t(j)]});
      cps[1].push_back({host::transpose(n2), &nt[size_t(j)]});
    }
    for (int side = 0; side < 2; ++side) {
      // right-hand side F f2 / C c2 (n x r), host
      const std::vector<double>& src = side == 0 ? B : Cc;
      const Mat& coef = side == 0 ? f2 : c2;
      const int cols = side == 0 ? m : q;
      std::vector<double> rhs(size_t(n) * r, 0.0);
      for (int c = 0; c < r; ++c)
        for (int t = 0; t < cols; ++t) {
          const double w = coef(t, c);
          if (w == 0.0) continue;
          for (int64_t i = 0; i < n; ++i) rhs[size_t(c) * n + size_t(i)] += src[size_t(t) * n + size_t(i)] * w;
        }
      double bn = 0.0;
      for (double v : rhs) bn += v * v;
      if (bn == 0.0)
        throw SolverError(std::string("birka: zero right-hand side on the ") + (side == 0 ? "trial" : "test") +
                          " side (sweep " + std::to_string(z) + "); input/output maps must be nonzero");
      int64_t estimate = 0;
      CsrPtr A = assemble_kron(dev, spec.blocks, side == 0 ? kh : kt, cps[side], estimate);
      mpg_report_row row{};
      row.sweep = z;
      row.point = side + 1;
      row.kind = MPG_KIND_NONE;
      row.min_residual = row.matrix_change = row.standard_residual = std::nan("");
      Side& sd = sides[side];
      if (cfg.mode != MPG_PRECOND_NONE && !sd.degraded && estimate > explicit_nnz_cap) {
        sd.degraded = true;
        out.warnings.push_back(std::string(side == 0 ? "trial" : "test") +
                               " side continues unpreconditioned: explicit operator assembly needs about " +
                               std::to_string(estimate) + " entries, above the cap of " +
                               std::to_string(explicit_nnz_cap) +
                               "; rerun with a fresh approximate inverse per sweep or without preconditioning");
      }
      ChainPtr prec;
      if (cfg.mode != MPG_PRECOND_NONE && !sd.degraded) {
        if (cfg.mode == MPG_PRECOND_REUSE_FROZEN && sd.chain) {
          row.kind = MPG_KIND_REUSED_SAME_MATRIX;
        } else if (cfg.mode == MPG_PRECOND_FRESH || cfg.mode == MPG_PRECOND_REUSE_FROZEN || !sd.chain || sd.chain->length() + 1 > cfg.max_chain_len) {
          SpaiOutcome so = spai_or_update(A, nullptr, cfg.spai, false);
          auto ch = std::make_shared<Chain>();
          ch->factors.push_back(so.p);
          sd.chain = ch;
          row.kind = MPG_KIND_FRESH;
          row.build_seconds = so.build_seconds;
        } else {
          SpaiOutcome so = spai_or_update(A, sd.prev, cfg.spai, false);
          auto ch = std::make_shared<Chain>(*sd.chain);
          ch->factors.push_back(so.p);
          sd.chain = ch;
          row.kind = MPG_KIND_VERTICAL;
          row.build_seconds = so.build_seconds;
          row.min_residual = so.min_residual;
          row.matrix_change = so.matrix_change;
        }
        if (cfg.mode == MPG_PRECOND_REUSE_CHAIN) sd.prev = A;
        prec = sd.chain;
        if (A->nrows <= cfg.standard_residual_max_dim) row.standard_residual = std_residual(A, prec);
      }
      OpPtr op = op_create(A, nullptr);
      std::vector<SolveSpec> specs(1);
      specs[0].sre = 0.0;
      specs[0].ca = 1.0;
      specs[0].chain = prec;
      specs[0].b = rhs.data();
      specs[0].x = side == 0 ? X.get() : Y.get();
      const GmresOutcome o = gmres_batch(*op, specs, cfg.gmres)[0];
      row.solves = 1;
      row.iterations = o.iterations;
      row.gmres_seconds = o.solve_seconds;
      out.rows.push_back(row);
      if (!o.converged) {
        char rel[32];
        std::snprintf(rel, sizeof rel, "%.3e", o.final_residual / std::max(o.rhs_norm, 1e-300));
        throw SolverError(std::string("birka: gmres did not converge on the ") + (side == 0 ? "trial" : "test") +
                          " side (sweep " + std::to_string(z) + "; relative residual " + rel + " after " +
                          std::to_string(o.iterations) + " iterations)");
      }
    }
    orthonormalize(dev, X.get(), n, r);
    orthonormalize(dev, Y.get(), n, r);
    const Mat wtv = ts_gram(dev, Y.get(), n, r, X.get(), n, r, n);
    host::LU lu(wtv);
    if (!lu.invertible())
      throw SolverError("birka: projection matrix (test basis^T trial basis) is singular at sweep " + std::to_string(z));
    for (int j = 0; j < r; ++j) {
      launch_spmv(*kp, X.get() + size_t(n) * j, T.get() + size_t(n) * j, 1.0, s);
      count_launch();
    }
    kr = lu.solve(ts_gram(dev, Y.get(), n, r, T.get(), n, r, n));
    for (int jn = 0; jn < m; ++jn) {
      for (int j = 0; j < r; ++j) {
        launch_spmv(*n_ops[size_t(jn)], X.get() + size_t(n) * j, T.get() + size_t(n) * j, 1.0, s);
        count_launch();
      }
      nr[size_t(jn)] = lu.solve(ts_gram(dev, Y.get(), n, r, T.get(), n, r, n));
    }
    fr = lu.solve(ts_gram(dev, Y.get(), n, r, Bd.get(), n, m, n));
    cr = ts_gram(dev, X.get(), n, r, Cd.get(), n, q, n);
    out.sweeps = z;
    const std::vector<host::Eig> lambda_new = host::sorted_eigenvalues(kr);
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < lambda_new.size(); ++i) {
      const double dr = lambda_new[i].re - lambda_prev[i].re, di = lambda_new[i].im - lambda_prev[i].im;
      num += dr * dr + di * di;
      den += lambda_prev[i].re * lambda_prev[i].re + lambda_prev[i].im * lambda_prev[i].im;
    }
    if (std::sqrt(num) / std::max(std::sqrt(den), 1e-300) < cfg.tol) out.converged = true;
    lambda_prev = lambda_new;
  }
  out.kr = kr;
  out.nr = nr;
  out.fr = fr;
  out.cr = cr;
  out.lambda = lambda_prev;
  out.v.resize(size_t(n) * r);
  out.w.resize(size_t(n) * r);
  MPG_CUDA(cudaMemcpyAsync(out.v.data(), X.get(), out.v.size() * 8, cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaMemcpyAsync(out.w.data(), Y.get(), out.w.size() * 8, cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  if (!out.converged)
    out.warnings.push_back("fixed point left unconverged after " + std::to_string(out.sweeps) + " sweeps");
  return out;
}

}  // namespace mpg
