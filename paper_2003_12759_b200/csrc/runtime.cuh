// Device runtime shared by all translation units of libmpg.so.
//
// Data layout in HBM:
//   * matrices: CSR with int32 row offsets and column indices, fp64 values;
//     a matrix's transpose (the reference's CSC shadow, sparse.cpp:27-46) is
//     a second CSR built on the device on first use;
//   * E sharing A's pattern is stored as interleaved (a, e) double2 pairs so
//     the fused shifted SpMV reads both with one 128-bit load per entry;
//   * Krylov bases live in 64-vector panels, each vector padded to a multiple
//     of 32 doubles (16-byte aligned double2 access).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mpg.h"

namespace mpg {

struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolverError : std::runtime_error { using std::runtime_error::runtime_error; };

#define MPG_CUDA(call)                                                                             \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw ::mpg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " __FILE__); \
  } while (0)

// Per-kernel-class profile (CUDA-event times + algorithmic bytes), filled by
// gmres_batch when profiling is enabled (mpg_profile_enable).
enum ProfKind {
  PK_CHAIN = 0, PK_OP, PK_DOT, PK_UPDPROBE, PK_UPD, PK_PROBE, PK_REORTH, PK_SMALL, PK_ASM, PK_COUNT
};
bool profile_enabled();
void profile_add(int kind, double ms, long long launches);
void profile_add_bytes(int kind, double bytes);

extern std::atomic<long long> g_launches;
inline void count_launch(long long k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
#define MPG_CHECK_LAUNCH() MPG_CUDA(cudaGetLastError())

// Per-device library context: one stream; allocations go through the
// stream-ordered pool (cudaMallocAsync) which doubles as the caching allocator.
struct DeviceCtx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
};
DeviceCtx& ctx(int device);

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) { cudaGetDevice(&prev); MPG_CUDA(cudaSetDevice(dev)); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void* dmalloc(int device, size_t bytes);
void dfree(int device, void* p);

template <class T>
struct DBuf {
  int device = 0;
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(int dev, size_t count) : device(dev), p(count ? static_cast<T*>(dmalloc(dev, count * sizeof(T))) : nullptr), n(count) {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : device(o.device), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { reset(); device = o.device; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() { if (p) dfree(device, p); p = nullptr; n = 0; }
  T* get() const { return p; }
};

// Row bins (the long-row split of irregular matrices, e.g. the C5 Zipf rows of
// 3 ... 2 000 entries): rows grouped by length class, class b served by
// sub-warps of 2 << b lanes (2, 4, 8, 16, 32), so a 2 000-entry row gets a
// whole warp and coalesced 256-byte value requests while the short rows keep
// 2-4 lanes. brow lists the rows class by class in ascending row order (a
// stable sort: deterministic, no atomics in the SpMV); boff[b] is class b's
// first slot in brow and bblk[b] its first 256-thread block, bblk[NBIN] the
// grid. Built with the matrix when max_row is far above the mean (spmv.cu).
constexpr int NBIN = 5;
__host__ __device__ __forceinline__ int row_bin(int len) {
  return len <= 5 ? 0 : len <= 32 ? 1 : len <= 64 ? 2 : len <= 128 ? 3 : 4;
}

// Kernel-side view of a CSR matrix.
struct CsrView {
  const int* rowptr;
  const int* colind;
  const double* val;
  int nrows, ncols;
  const int* brow;  // null: no row bins
  int boff[NBIN + 1];
  int bblk[NBIN + 1];
};

#ifdef __CUDACC__
// Binned thread mapping: this thread's row (or ok = false), sub-warp width and lane.
__device__ __forceinline__ bool bin_locate(const CsrView& f, int& row, int& W, int& lane) {
  int b = 0;
#pragma unroll
  for (int i = 1; i < NBIN; ++i) b += int(blockIdx.x) >= f.bblk[i];
  W = 2 << b;
  const int t = (int(blockIdx.x) - f.bblk[b]) * int(blockDim.x) + int(threadIdx.x);
  const int slot = t >> (b + 1);
  lane = t & (W - 1);
  row = 0;
  if (slot >= f.boff[b + 1] - f.boff[b]) return false;
  row = f.brow[f.boff[b] + slot];
  return true;
}
__device__ __forceinline__ double sub_sum_rt(double v, int W) {
  for (int o = W >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
  return v;
}
#endif

// Halo-staged sliced ELL (spmv.cu halo_*; the multi-RHS SpMV of the run-mode
// groups in gmres.cu). Rows in blocks of HALO_R; per block the sorted unique
// columns its rows touch (the halo, staged once into shared memory per SpMV)
// and, per 32-row slice, the entries column-major (entry j of lane l at
// sptr[slice] + 32 j + l) with 16-bit local indices into the block's halo.
// The matrix stream is then 2 B of index + the value per entry, coalesced, and
// the x-gather reads shared memory instead of L1/L2. Built once per pattern on
// the device; a pattern whose blocks exceed HALO_MAXNZ entries or HALO_MAX
// halo columns gets none (the CSR kernels run instead).
constexpr int HALO_R = 128;
constexpr int HALO_MAX = 1536;
constexpr int HALO_MAXNZ = 8192;
constexpr int HALO_XSTRIDE = 4;  // double2 per staged x row; the 4 chunks are XOR-swizzled by (row >> 1) & 3
struct HaloPattern {
  int nrows = 0, nblocks = 0, max_halo = 0;
  int64_t entries = 0;
  DBuf<int> hoff, halo, sptr, perm;  // [nblocks + 1], [hoff.back()], [nslices + 1], [entries] (-1: padding)
  DBuf<unsigned short> lidx;         // [entries]
};
using HaloPatternPtr = std::shared_ptr<const HaloPattern>;
struct HaloView {
  int nrows;
  const int* hoff;
  const int* halo;
  const int* sptr;
  const unsigned short* lidx;
  const double* val;    // one value per entry (a matrix or factor)
  const double2* val2;  // (a, e) per entry (E sharing A's pattern)
};
struct DevCsr;
HaloPatternPtr halo_pattern_build(const DevCsr& m);  // nullptr if the pattern does not fit

// Sliced ELL with 8-row slices (SELL-8) for the interleaved multi-RHS SpMVs:
// entry j of row r sits at sptr[r / 8] + 8 j + r % 8, so the 8 rows a warp
// covers (4 lanes per row) load their column index and value of step j from 8
// consecutive slots -- one request each instead of 8 scattered ones (the CSR
// kernels are L1-wavefront bound on those, not on DRAM). Padding: index of the
// row itself, value 0. Built once per pattern (nullptr: padding > 25 %).
struct Sell8 {
  int nrows = 0;
  int64_t entries = 0;
  int max_tile = 0;  // most entries in a block of 8 consecutive slices (k_spmv_sell8t's shared-memory tile)
  DBuf<int> sptr, col, perm;  // [nslices + 1], [entries], [entries] (-1: padding)
};
using Sell8Ptr = std::shared_ptr<const Sell8>;
struct Sell8View {
  int nrows;
  const int* sptr;
  const int* col;
  const double* val;
  const double2* val2;
};
Sell8Ptr sell8_build(const DevCsr& m);

struct DevCsr {
  int device = 0;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  DBuf<int> rowptr, colind;
  DBuf<double> val;
  int max_row = 0;     // longest row
  double mean_row = 0; // nnz / nrows
  bool is_diag = false;
  mutable std::mutex mu;
  mutable std::shared_ptr<DevCsr> tcache;  // transpose, built on first use
  mutable bool halo_tried = false;          // halo pattern + this matrix's values in it, built on first use
  mutable HaloPatternPtr halo;
  mutable DBuf<double> halo_val;
  mutable bool sell_tried = false;          // SELL-8 layout + this matrix's values in it, built on first use
  mutable Sell8Ptr sell;
  mutable DBuf<double> sell_val;
  DBuf<int> brow;  // row bins (CsrView): empty for regular matrices
  int boff[NBIN + 1] = {}, bblk[NBIN + 1] = {};
  CsrView view() const {
    CsrView v{rowptr.get(), colind.get(), val.get(), int(nrows), int(ncols), brow.get(), {}, {}};
    for (int i = 0; i <= NBIN; ++i) { v.boff[i] = boff[i]; v.bblk[i] = bblk[i]; }
    return v;
  }
};
// The halo layout of m with m's own values (nullptr: not eligible); cached on m.
const HaloPattern* halo_of(const DevCsr& m, HaloView* view);
// The SELL-8 layout of m with m's own values (nullptr: not eligible); cached on m.
const Sell8* sell_of(const DevCsr& m, Sell8View* view);
using CsrPtr = std::shared_ptr<DevCsr>;

// Builders (spmv.cu).
CsrPtr csr_from_host(int device, int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci, const double* v);
CsrPtr csr_from_device_parts(int device, int64_t nr, int64_t nc, DBuf<int>&& rp, DBuf<int>&& ci, DBuf<double>&& v);
CsrPtr csr_transpose(const DevCsr& a);           // deterministic counting-sort transpose
CsrPtr csr_transpose_cached(const CsrPtr& a);
void csr_finalize_stats(DevCsr& m);              // max_row / mean_row / is_diag (syncs)

// Shifted operator family sigma E - A.
enum EMode { E_IDENT = 0, E_DIAG = 1, E_SAMEPAT = 2, E_GENERAL = 3 };
struct OpView {
  CsrView a;
  int emode;
  const double* ediag;  // E_DIAG
  const double2* ae;    // E_SAMEPAT: (a_k, e_k) along A's pattern
  CsrView e;            // E_GENERAL
};
struct ShiftedOp {
  int device = 0;
  int64_t n = 0;
  int emode = E_IDENT;
  CsrPtr a, e, at, et;
  DBuf<double> ediag;
  DBuf<double2> ae, ae_t;
  int vec_width = 32;  // sub-warp width for this operator's rows
  mutable std::mutex halo_mu;
  mutable bool halo_tried[2] = {false, false};
  mutable DBuf<double2> halo_ae[2];  // (a, e) in the halo layout of A / A^T (E_SAMEPAT)
  mutable bool sell_tried_op[2] = {false, false};
  mutable DBuf<double2> sell_ae[2];  // (a, e) in the SELL-8 layout of A / A^T (E_SAMEPAT)
  OpView view(bool transpose) const;
};
using OpPtr = std::shared_ptr<ShiftedOp>;
OpPtr op_create(const CsrPtr& a, const CsrPtr& e);
// The halo layout of the operator side (A's pattern; values of A, or (a, e)
// pairs for E_SAMEPAT); nullptr if not eligible.
const HaloPattern* halo_of_op(const ShiftedOp& op, bool transpose, HaloView* view);
const Sell8* sell_of_op(const ShiftedOp& op, bool transpose, Sell8View* view);

// Explicit unit matrix sigma E - A (or its 2n pair form) on the device.
CsrPtr op_explicit(const ShiftedOp& op, double sre, double sim, bool transpose);

// Immutable chain (base + factors), factors shared between chains.
struct Chain {
  std::vector<CsrPtr> factors;  // [0] = base
  int length() const { return int(factors.size()) - 1; }
};
using ChainPtr = std::shared_ptr<const Chain>;

int choose_vec_width(double mean_row);

// ---- launches (spmv.cu) ------------------------------------------------------
// y = alpha * M x
void launch_spmv(const DevCsr& m, const double* x, double* y, double alpha, cudaStream_t s);
// y = scale * (sigma E - A) x   (pair form when sim != 0: x, y have 2n entries)
// resid != null: y = resid - (sigma E - A) x
void launch_op(const ShiftedOp& op, bool transpose, double sre, double sim, double ca, const double* x, double* y,
               const double* resid, double scale, cudaStream_t s, double* tmp_general);
// y = Q_L(...Q_1(P x)); tmp must hold n doubles.
void launch_chain(const Chain& c, const double* x, double* y, double* tmp, cudaStream_t s);
double device_norm2(int device, const double* x, int64_t n, cudaStream_t s);

// Host <-> any memory helpers.
bool is_device_ptr(const void* p);
void copy_in(double* dst_dev, const double* src_any, size_t n, cudaStream_t s);
void copy_out(double* dst_any, const double* src_dev, size_t n, cudaStream_t s);

// ---- GMRES (gmres.cu) --------------------------------------------------------
struct SolveSpec {
  double sre = 0, sim = 0;
  bool transpose = false;
  double ca = -1.0;         // -1: sigma E - A;  +1 (with sigma = 0, E = I): plain A
  ChainPtr chain;           // null: identity
  bool pair_blockdiag = false;  // apply an n x n chain blockwise on a 2n pair vector
  const double* b = nullptr;    // any memory
  double* x = nullptr;          // any memory
};
struct GmresOptions { double rel_tol = 1e-6; int max_iter = 1000; bool record_history = false; };
struct GmresOutcome {
  int iterations = 0;
  bool converged = false, breakdown = false;
  double rhs_norm = 0, final_residual = 0, solve_seconds = 0;
  int reorth_passes = 0;
  std::vector<double> history;
};
std::vector<GmresOutcome> gmres_batch(const ShiftedOp& op, std::vector<SolveSpec>& specs, const GmresOptions& opt);

// ---- SPAI (spai.cu) ------------------------------------------------------------
struct SpaiOptions {
  int pattern_kind = 1, power = 2;
  double fill_tol = 1e-4;
  int max_fill_per_col = 50, max_pattern_sweeps = 3;
};
struct SpaiOutcome {
  CsrPtr p;
  std::vector<double> column_residuals;  // host
  int64_t fallback_count = 0;
  double build_seconds = 0;
  double min_residual = 0, matrix_change = 0;  // update builds
};
// prev == nullptr: spai_build (rhs = e_col); else update_build (rhs = prev(:, col)).
SpaiOutcome spai_or_update(const CsrPtr& a, const CsrPtr& prev, const SpaiOptions& o, bool want_residuals);
double frobenius_distance(const CsrPtr& a, const CsrPtr& b);
void spai_column_solve_dev(const CsrPtr& a, int64_t col, const std::vector<int64_t>& pattern, std::vector<double>& values,
                           double& residual, bool& rank_def);

}  // namespace mpg
