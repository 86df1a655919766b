// K2 + K3: device-resident, multi-shift batched GMRES
// (gmres_right_preconditioned, proj/src/gmres.cpp:40-186).
//
// Control flow follows the reference step by step, per solve:
//   v0 = b/||b|| (:46-55); per iteration P then A (:96-97); Gram-Schmidt
//   (:101-105, here the classical form with one fused read of the basis per
//   pass); the measured second pass when ||V^T w|| > 1e-10 ||w|| (:108-119);
//   invariance at 1e-14 ||w_pre|| (:121-122); Givens (:125-157); lucky
//   breakdown (:159-164); the true-residual recheck with the 0.25 back-off
//   (:166-180); finish with a recomputed residual (:81-93).
// All scalar control runs on the device; the host launches the captured
// iteration graph in chunks and polls the solve phases once per chunk.
//
// Basis vectors are stored unnormalised with a per-vector scale s_j =
// 1/||w_j|| (v_j = s_j W_j), which removes the normalisation pass; the
// preconditioner and operator are linear, so P v_k = s_k (P W_k).
//
// Roofline: per iteration B_S + B_P + 16 (k+1) n + 32 n bytes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "runtime.cuh"

namespace mpg {
namespace {

constexpr int PH_RUN = 0, PH_ASM = 1, PH_DONE = 2;
constexpr int ASM_RECHECK = 1, ASM_FINISH = 2;
constexpr int DOT_TILE = 1024;   // rows per tile of the dot kernel
constexpr int UPD_TILE = 512;    // rows per tile of the update kernel (256 threads x double2)
constexpr int PANEL = 64;        // basis vectors per allocation panel
// Basis layout: 64-vector panels stored chunk-major, [ld / CHUNK][64][CHUNK]:
// the CHUNK = 16 rows (128 B) of the 64 vectors of a panel form one contiguous
// 8 KB block. The Gram-Schmidt passes walk tiles of T rows x (k+1) vectors;
// with plain vectors a tile touches k+1 distinct 2 MB pages (one per vector)
// and ran at 4.6 TB/s for 16-row tiles, chunk-major it touches ceil((k+1)/64)
// contiguous blocks (scripts/membench.cu: 5.8-6.6 TB/s for the same walk).
// V[j] points at the vector's first chunk (panel + (j % 64) * CHUNK); row r of
// it is V[j][vidx(r)]. Pairs of rows (r even) are contiguous.
constexpr int CHUNK = 16;
__host__ __device__ __forceinline__ int vidx(int r) { return (r / CHUNK) * (PANEL * CHUNK) + (r % CHUNK); }

struct GmSolve {
  // configuration
  int n, nbase, pair, transpose, stages, pair_bd, max_iter, record;
  double sre, sim, ca, target, bnorm;
  // state
  int k, phase, asm_kind, asm_k, guess, iterations, converged, breakdown, xsel, reorth_count;
  int grouped_op;     // bit 0: run-mode operator by a group kernel, bit 1: assembly-mode
  int grouped_chain;  // handled by the shared-matrix (multi-RHS) kernels
  int il_run;         // complex pair riding in an interleaved group as two columns: run-mode chain by the group kernels
  int dcgs;           // delayed second pass enabled (fused path)
  int pend;           // V[k] awaits its second-pass correction V[k] -= sum_j dp_j s_j V_j (DCGS2)
  double estimate, recheck_at, w2_pre, w2_a, w2_b, wn_cur, final_residual;
  // arrays
  double** V;
  double* scale;
  double* h;
  double* d;
  double* H;
  double* cs;
  double* sn;
  double* g;
  double* hist;
  double* y;
  double* z0;
  double* z1;
  double* ubuf;
  double* rbuf;
  double* part;
  const CsrView* fac;
  const CUtensorMap* tm;  // per basis panel: [2 p] 64-vector box, [2 p + 1] 8-vector box (null: none)
  double* dp;  // pending second-pass coefficients (the previous iteration's probe d)
  double* hg;  // this iteration's Hessenberg column (h holds the update coefficients)
  double* Hu;  // unrotated Hessenberg columns, column i at hoff2(i), i + 2 entries
  float** F;   // single-precision shadow of the basis (null: none): F[j] row r at fidx(r)
  const CUtensorMap* tmf;  // per shadow panel: [2 p] 64-vector box, [2 p + 1] 8-vector box
};
__host__ __device__ __forceinline__ size_t hoff2(int i) { return size_t(i) * size_t(i + 3) / 2; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int V>
__device__ __forceinline__ double sub_sum(double v) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, V);
  return v;
}

__device__ __forceinline__ size_t hoff(int j) { return size_t(j) * size_t(j + 1) / 2; }

// ---- chain stage: z[stage&1] = F_stage * src ------------------------------------
// Irregular (row-binned) factors gather x at random columns: the chunk-major basis
// vector V[k] (one 8 KB panel block per 16 rows: a 1 GB span at n = 2 M) is copied
// to the plain vector z1 first, which stage 0 then reads (C5: chain SpMV 683 us with
// the chunk-major gather against 326 us for the same-sized operator on a plain vector).
__global__ void __launch_bounds__(256) k_unchunk(GmSolve* S, const int* __restrict__ list) {
  GmSolve& st = S[list[blockIdx.y]];
  if (st.phase != PH_RUN || st.stages == 0 || st.grouped_chain || st.il_run) return;
  if (!st.fac[0].brow) return;
  const double* v = st.V[st.k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += gridDim.x * blockDim.x) st.z1[i] = v[vidx(i)];
}

// V = 0: the row-binned mapping for irregular factors (runtime.cuh bin_locate);
// a solve is served by the launch that matches its factor.
template <int V>
__global__ void __launch_bounds__(256) k_chain_stage(GmSolve* S, int stage, int mode, const int* __restrict__ list) {
  // list: the solves this launch serves (those not advanced by a group kernel in this mode); blockIdx.y walks it
  GmSolve& st = S[list[blockIdx.y]];
  if (mode == 0 ? st.phase != PH_RUN : st.phase != PH_ASM) return;
  if (stage >= st.stages || st.grouped_chain || (mode == 0 && st.il_run)) return;
  const CsrView f = st.fac[stage];
  if ((f.brow != nullptr) != (V == 0)) return;
  const int halves = st.pair_bd ? 2 : 1;
  const bool chunked = stage == 0 && mode == 0;  // reads the basis vector V[k]
  const double* src = stage == 0 ? (mode == 0 ? st.V[st.k] : st.ubuf) : ((stage - 1) & 1 ? st.z1 : st.z0);
  double* dst = (stage & 1) ? st.z1 : st.z0;
  if (V == 0) {
    if (int(blockIdx.x) >= f.bblk[NBIN]) return;
    int r, W, lane;
    const bool ok = bin_locate(f, r, W, lane);
    if (chunked) src = st.z1;  // k_unchunk's plain copy of V[k]
    for (int hf = 0; hf < halves; ++hf) {
      const int off = hf * f.nrows;
      double acc = 0.0;
      if (ok) {
        const int b = f.rowptr[r], e = f.rowptr[r + 1];
        const double* x = src + off;
#pragma unroll 4
        for (int k = b + lane; k < e; k += W) acc = fma(__ldcs(f.val + k), __ldg(x + __ldcs(f.colind + k)), acc);
      }
      acc = sub_sum_rt(acc, W);
      if (ok && lane == 0) dst[off + r] = acc;
    }
    return;
  }
  constexpr int VV = V ? V : 2;
  const int lane = threadIdx.x & (VV - 1);
  // grid-stride over row blocks (the assembly-mode launch uses a small grid: it is idle in almost every iteration)
  const int64_t rows_total = int64_t(f.nrows) * (halves == 2 ? 1 : halves);
  for (int64_t base = int64_t(blockIdx.x) * (256 / VV); base < rows_total; base += int64_t(gridDim.x) * (256 / VV)) {
  const int row = int(base) + int(threadIdx.x) / VV;
  if (halves == 2) {
    // complex pair, block-diagonal factor: both halves from one pass over the factor's row
    // (the factor was read once per half: 0.4 -> 0.25 ms per pair solve and iteration on C3)
    double a0 = 0.0, a1 = 0.0;
    const int nr = f.nrows;
    if (row < nr) {
      const int b = f.rowptr[row], e = f.rowptr[row + 1];
#pragma unroll 4
      for (int k = b + lane; k < e; k += VV) {
        const double fv = __ldcs(f.val + k);
        const int c = __ldcs(f.colind + k);
        a0 = fma(fv, __ldg(src + (chunked ? vidx(c) : c)), a0);
        a1 = fma(fv, __ldg(src + (chunked ? vidx(nr + c) : nr + c)), a1);
      }
    }
    a0 = sub_sum<VV>(a0);
    a1 = sub_sum<VV>(a1);
    if (row < nr && lane == 0) {
      dst[row] = a0;
      dst[nr + row] = a1;
    }
    continue;
  }
  double acc = 0.0;
  int r = row, off = 0;
  if (row >= f.nrows) { r = row - f.nrows; off = f.nrows; }
  if (row < f.nrows * halves) {
    const int b = f.rowptr[r], e = f.rowptr[r + 1];
    if (chunked) {
#pragma unroll 4
      for (int k = b + lane; k < e; k += VV)
        acc = fma(__ldcs(f.val + k), __ldg(src + vidx(off + __ldcs(f.colind + k))), acc);
    } else {
      const double* x = src + off;
#pragma unroll 4
      for (int k = b + lane; k < e; k += VV) acc = fma(__ldcs(f.val + k), __ldg(x + __ldcs(f.colind + k)), acc);
    }
  }
  acc = sub_sum<VV>(acc);
  if (row < f.nrows * halves && lane == 0) dst[off + r] = acc;
  }
}

// ---- operator: W_{k+1} = s_k (sigma E - A) z  /  r = b - (sigma E - A) x ---------
template <int V, int EM>
__global__ void __launch_bounds__(256) k_iter_op(GmSolve* S, OpView opn, OpView opt, int mode,
                                                 const int* __restrict__ list) {
  GmSolve& st = S[list[blockIdx.y]];
  if (mode == 0 ? st.phase != PH_RUN : st.phase != PH_ASM) return;
  if (st.grouped_op & (mode == 0 ? 1 : 2)) return;
  const OpView& op = st.transpose ? opt : opn;
  if ((op.a.brow != nullptr) != (V == 0)) return;  // V = 0 serves the row-binned operator sides
  const int n = op.a.nrows;
  const double* x;
  if (mode == 0) x = st.stages ? ((st.stages - 1) & 1 ? st.z1 : st.z0) : st.V[st.k];
  else x = st.stages ? ((st.stages - 1) & 1 ? st.z1 : st.z0) : st.ubuf;
  // grid-stride over row blocks for the fixed-width mapping (small grids in assembly mode); one pass for V = 0
  constexpr int RPB = V ? 256 / (V ? V : 1) : 1;
  for (int64_t base = int64_t(blockIdx.x) * RPB;; base += int64_t(gridDim.x) * RPB) {
  if (V != 0 && base >= n) break;
  int lane, row, W = V;
  bool ok;
  if (V == 0) {
    if (int(blockIdx.x) >= op.a.bblk[NBIN]) return;
    ok = bin_locate(op.a, row, W, lane);
  } else {
    lane = threadIdx.x & (V - 1);
    row = int(base) + int(threadIdx.x) / (V ? V : 1);
    ok = row < n;
  }
  const bool xc = mode == 0 && st.stages == 0;  // x is a chunk-major basis vector
  const bool pair = st.pair;
  double a1 = 0.0, a2 = 0.0, e1 = 0.0, e2 = 0.0;
  if (ok) {
    const int b = op.a.rowptr[row], e = op.a.rowptr[row + 1];
    if (EM == E_SAMEPAT) {
#pragma unroll 4
      for (int k = b + lane; k < e; k += W) {
        const double2 ae = __ldcs(op.ae + k);
        const int c = __ldcs(op.a.colind + k);
        const double x1 = __ldg(x + (xc ? vidx(c) : c));
        a1 = fma(ae.x, x1, a1);
        e1 = fma(ae.y, x1, e1);
        if (pair) {
          const double x2 = __ldg(x + (xc ? vidx(n + c) : n + c));
          a2 = fma(ae.x, x2, a2);
          e2 = fma(ae.y, x2, e2);
        }
      }
    } else {
#pragma unroll 4
      for (int k = b + lane; k < e; k += W) {
        const double av = __ldcs(op.a.val + k);
        const int c = __ldcs(op.a.colind + k);
        a1 = fma(av, __ldg(x + (xc ? vidx(c) : c)), a1);
        if (pair) a2 = fma(av, __ldg(x + (xc ? vidx(n + c) : n + c)), a2);
      }
    }
  }
#define MPG_SUBSUM(v) v = V ? sub_sum<(V ? V : 2)>(v) : sub_sum_rt(v, W)
  MPG_SUBSUM(a1);
  MPG_SUBSUM(a2);
  if (EM == E_SAMEPAT) {
    MPG_SUBSUM(e1);
    MPG_SUBSUM(e2);
  }
#undef MPG_SUBSUM
  if (ok && lane == 0) {
    const int i1 = xc ? vidx(row) : row, i2 = xc ? vidx(n + row) : n + row;
    if (EM == E_IDENT) {
      e1 = x[i1];
      if (pair) e2 = x[i2];
    } else if (EM == E_DIAG) {
      const double dd = op.ediag[row];
      e1 = dd * x[i1];
      if (pair) e2 = dd * x[i2];
    }
    const double sre = st.sre, sim = st.sim, ca = st.ca;
    double y1, y2 = 0.0;
    if (pair) {
      y1 = sre * e1 + ca * a1 + sim * e2;
      y2 = -sim * e1 + sre * e2 + ca * a2;
    } else {
      y1 = sre * e1 + ca * a1;
    }
    if (mode == 0) {
      double* w = st.V[st.k + 1];
      const double sc = st.scale[st.k];
      w[vidx(row)] = sc * y1;
      if (pair) w[vidx(n + row)] = sc * y2;
    } else {
      const double* b0 = st.V[0];
      st.rbuf[row] = b0[vidx(row)] - y1;
      if (pair) st.rbuf[n + row] = b0[vidx(n + row)] - y2;
    }
  }
  if (V == 0) break;
  }
}

// ---- shared-matrix (multi-RHS) variants ----------------------------------------
// Solves of a batch that apply the same matrix — the same chain factor (a
// frozen or shared preconditioner) or the same side of the operator (all
// primal or all dual real shifts) — are advanced by one launch that reads
// each matrix entry once and applies it to up to MB right-hand sides: the
// matrix bytes are paid once per group instead of once per solve.
constexpr int MB = 8;

// half: 0 a real solve's column; 1 / 2 the two halves of a complex pair (2n real form) that rides in the
// group as two adjacent columns starting at an even one: the preconditioner is block diagonal and the
// operator's A x and E x are per column, only the epilogue couples them (k_spmv_sell8t).
struct Group {
  int idx[MB];
  int cnt;
  unsigned hm;  // two bits per column (a register, not an indexed parameter array)
  __host__ __device__ int half(int q) const { return int((hm >> (2 * q)) & 3u); }
  __host__ __device__ void set_half(int q, int h) { hm = (hm & ~(3u << (2 * q))) | (unsigned(h) << (2 * q)); }
};

template <int V>
__global__ void __launch_bounds__(256) k_chain_multi(GmSolve* S, Group grp, CsrView f, int stage, int mode) {
  const bool basis = stage == 0 && mode == 0;  // reading V[k] (chunk-major)
  const double* src[MB];
  double* dst[MB];
  bool act[MB];
  bool any = false;
#pragma unroll
  for (int q = 0; q < MB; ++q) {
    act[q] = false;
    src[q] = nullptr;
    dst[q] = nullptr;
    if (q < grp.cnt) {
      const GmSolve& st = S[grp.idx[q]];
      act[q] = (mode == 0 ? st.phase == PH_RUN : st.phase == PH_ASM) && stage < st.stages;
      src[q] = stage == 0 ? (mode == 0 ? st.V[st.k] : st.ubuf) : ((stage - 1) & 1 ? st.z1 : st.z0);
      dst[q] = (stage & 1) ? st.z1 : st.z0;
      any |= act[q];
    }
  }
  if (!any) return;
  const int lane = threadIdx.x & (V - 1);
  // grid-stride over row blocks (small grids for the mostly idle assembly-mode launches, see k_iter_op_multi)
  for (int64_t base = int64_t(blockIdx.x) * (256 / V); base < f.nrows; base += int64_t(gridDim.x) * (256 / V)) {
    const int row = int(base) + int(threadIdx.x) / V;
    double acc[MB];
#pragma unroll
    for (int q = 0; q < MB; ++q) acc[q] = 0.0;
    if (row < f.nrows) {
      const int b = f.rowptr[row], e = f.rowptr[row + 1];
#pragma unroll 2
      for (int k = b + lane; k < e; k += V) {
        const double a = __ldcs(f.val + k);
        const int c = __ldcs(f.colind + k);
#pragma unroll
        for (int q = 0; q < MB; ++q)
          if (act[q]) acc[q] = fma(a, __ldg(src[q] + (basis ? vidx(c) : c)), acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) acc[q] = sub_sum<V>(acc[q]);
    if (row < f.nrows && lane == 0) {
#pragma unroll
      for (int q = 0; q < MB; ++q)
        if (act[q]) dst[q][row] = acc[q];
    }
  }
}

template <int V, int EM>
__global__ void __launch_bounds__(256) k_iter_op_multi(GmSolve* S, Group grp, OpView op, int mode) {
  const double* xs[MB];
  bool xb[MB];  // x is the basis vector V[k] (no chain)
  bool act[MB];
  bool any = false;
#pragma unroll
  for (int q = 0; q < MB; ++q) {
    act[q] = false;
    xs[q] = nullptr;
    xb[q] = false;
    if (q < grp.cnt) {
      const GmSolve& st = S[grp.idx[q]];
      act[q] = mode == 0 ? st.phase == PH_RUN : st.phase == PH_ASM;
      if (mode == 0) xs[q] = st.stages ? ((st.stages - 1) & 1 ? st.z1 : st.z0) : st.V[st.k];
      else xs[q] = st.stages ? ((st.stages - 1) & 1 ? st.z1 : st.z0) : st.ubuf;
      xb[q] = mode == 0 && st.stages == 0;
      any |= act[q];
    }
  }
  if (!any) return;
  const int n = op.a.nrows;
  const int lane = threadIdx.x & (V - 1);
  // grid-stride over row blocks: the assembly-mode launches (one per iteration in the captured graph,
  // almost always with no solve in assembly) use a small grid, so an idle launch costs a few
  // microseconds instead of the ~50 us of 18 600 CTAs that each read the solve states and exit
  for (int64_t base = int64_t(blockIdx.x) * (256 / V); base < n; base += int64_t(gridDim.x) * (256 / V)) {
  const int row = int(base) + int(threadIdx.x) / V;
  double a1[MB], e1[MB];
#pragma unroll
  for (int q = 0; q < MB; ++q) a1[q] = e1[q] = 0.0;
  if (row < n) {
    const int b = op.a.rowptr[row], e = op.a.rowptr[row + 1];
#pragma unroll 2
    for (int k = b + lane; k < e; k += V) {
      const int c = __ldcs(op.a.colind + k);
      if (EM == E_SAMEPAT) {
        const double2 ae = __ldcs(op.ae + k);
#pragma unroll
        for (int q = 0; q < MB; ++q)
          if (act[q]) {
            const double xv = __ldg(xs[q] + (xb[q] ? vidx(c) : c));
            a1[q] = fma(ae.x, xv, a1[q]);
            e1[q] = fma(ae.y, xv, e1[q]);
          }
      } else {
        const double av = __ldcs(op.a.val + k);
#pragma unroll
        for (int q = 0; q < MB; ++q)
          if (act[q]) a1[q] = fma(av, __ldg(xs[q] + (xb[q] ? vidx(c) : c)), a1[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < MB; ++q) {
    a1[q] = sub_sum<V>(a1[q]);
    if (EM == E_SAMEPAT) e1[q] = sub_sum<V>(e1[q]);
  }
  if (row < n && lane == 0) {
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      if (!act[q]) continue;
      GmSolve& st = S[grp.idx[q]];
      double ex = e1[q];
      const int xr = xb[q] ? vidx(row) : row;
      if (EM == E_IDENT) ex = xs[q][xr];
      else if (EM == E_DIAG) ex = op.ediag[row] * xs[q][xr];
      const double y1 = st.sre * ex + st.ca * a1[q];
      if (mode == 0) st.V[st.k + 1][vidx(row)] = st.scale[st.k] * y1;
      else st.rbuf[row] = st.V[0][vidx(row)] - y1;
    }
  }
  }
}

// ---- interleaved multi-RHS path (run mode) --------------------------------------
// A group whose solves share the chain AND the operator side keeps its MB
// right-hand sides interleaved, x[row][q] (64 B per row): a gather of column c
// then fetches all MB values with four 128-bit loads from one 64-byte span
// instead of MB separate 8-byte gathers (4x fewer L1/L2 sectors; the separate
// gathers made the shared-matrix SpMVs L1/latency bound at ~1.5-2 TB/s of
// DRAM traffic, profiles/r01/ncu_full_c3_summary.txt).
// Narrow mode: once at most MBN = 4 real columns of a group are still running (the solves of an IRKA sweep
// converge after 80 ... 320 iterations: three quarters of a group's iterations run with <= 4 columns) the
// interleave shrinks to x[row][4] and each of a row's four lanes carries one right-hand side, so the
// x-gather, which bounds these kernels through the L1 data pipe, moves 32 instead of 64 bytes per nonzero.
// Every kernel of the path derives the mode and the slot -> column map from the solve phases, which only
// k_finalize changes, and branches (uniformly over the grid) into the wide or the narrow loop. Groups with a
// running complex pair stay wide. Bit 31 of hm allows the mode.
constexpr int MBN = 4;
// The decision, by the first warp of a block, one solve state per lane (a single round trip instead of a
// chain of eight): md[0..3] the slots' columns (the running columns in order, -1 past them), md[4] narrow
// (allowed, at most MBN running, none of them half of a pair), md[5] any column running.
__device__ __forceinline__ void il_mode_warp(const GmSolve* S, const Group& grp, int* md) {
  const int q = threadIdx.x & 31;
  int idx = 0;
#pragma unroll
  for (int u = 0; u < MB; ++u)
    if (u == q) idx = grp.idx[u];
  const bool run = q < grp.cnt && S[idx].phase == PH_RUN;
  const unsigned m = __ballot_sync(0xffffffffu, run);
  if (q == 0) {
    unsigned pm = 0;
#pragma unroll
    for (int u = 0; u < MB; ++u)
      if (grp.half(u)) pm |= 1u << u;
    unsigned r = m;
    for (int t = 0; t < MBN; ++t) {
      md[t] = r ? __ffs(r) - 1 : -1;
      r &= r - 1;
    }
    md[4] = ((grp.hm >> 31) && __popc(m) <= MBN && !(m & pm)) ? 1 : 0;
    md[5] = m != 0 ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256) k_pack_il(GmSolve* S, Group grp, double* xa, int n) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  __shared__ int md[6];  // the first warp reads the solve states for the block
  if (threadIdx.x < 32) il_mode_warp(S, grp, md);
  __syncthreads();
  const int q0 = md[0], q1 = md[1], q2 = md[2], q3 = md[3];
  if (md[4]) {
    const int row = int(i / MBN), t = int(i % MBN);
    if (row >= n) return;
    const int q = t == 0 ? q0 : t == 1 ? q1 : t == 2 ? q2 : q3;
    double v = 0.0;
    if (q >= 0) {
      const GmSolve& st = S[grp.idx[q]];
      v = st.V[st.k][vidx(row)];
    }
    xa[i] = v;
    return;
  }
  const int row = int(i / MB), q = int(i % MB);
  if (row >= n) return;
  double v = 0.0;
  if (q < grp.cnt) {
    const GmSolve& st = S[grp.idx[q]];
    if (st.phase == PH_RUN) v = st.V[st.k][vidx(grp.half(q) == 2 ? n + row : row)];
  }
  xa[i] = v;
}

__device__ __forceinline__ bool il_any_run(const GmSolve* S, const Group& grp) {
  bool any = false;
  for (int q = 0; q < grp.cnt; ++q) any |= S[grp.idx[q]].phase == PH_RUN;
  return any;
}

template <int V>
__global__ void __launch_bounds__(256) k_chain_il(GmSolve* S, Group grp, CsrView f, const double* __restrict__ xin,
                                                  double* __restrict__ xout) {
  if (!il_any_run(S, grp)) return;
  const int lane = threadIdx.x & (V - 1);
  const int row = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) / V);
  double acc[MB];
#pragma unroll
  for (int q = 0; q < MB; ++q) acc[q] = 0.0;
  if (row < f.nrows) {
    const int b = f.rowptr[row], e = f.rowptr[row + 1];
#pragma unroll 2
    for (int k = b + lane; k < e; k += V) {
      const double a = __ldcs(f.val + k);
      const double2* xp = reinterpret_cast<const double2*>(xin + size_t(__ldcs(f.colind + k)) * MB);
#pragma unroll
      for (int h = 0; h < MB / 2; ++h) {
        const double2 x = __ldg(xp + h);
        acc[2 * h] = fma(a, x.x, acc[2 * h]);
        acc[2 * h + 1] = fma(a, x.y, acc[2 * h + 1]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < MB; ++q) acc[q] = sub_sum<V>(acc[q]);
  if (row < f.nrows) {
    double2* yp = reinterpret_cast<double2*>(xout + size_t(row) * MB);
#pragma unroll
    for (int h = 0; h < MB / 2; ++h)
      if (h % V == lane) yp[h] = make_double2(acc[2 * h], acc[2 * h + 1]);
  }
}

template <int V, int EM>
__global__ void __launch_bounds__(256) k_op_il(GmSolve* S, Group grp, OpView op, const double* __restrict__ xin) {
  if (!il_any_run(S, grp)) return;
  const int n = op.a.nrows;
  const int lane = threadIdx.x & (V - 1);
  const int row = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) / V);
  double a1[MB], e1[MB];
#pragma unroll
  for (int q = 0; q < MB; ++q) a1[q] = e1[q] = 0.0;
  if (row < n) {
    const int b = op.a.rowptr[row], e = op.a.rowptr[row + 1];
#pragma unroll 2
    for (int k = b + lane; k < e; k += V) {
      const double2* xp = reinterpret_cast<const double2*>(xin + size_t(__ldcs(op.a.colind + k)) * MB);
      if (EM == E_SAMEPAT) {
        const double2 ae = __ldcs(op.ae + k);
#pragma unroll
        for (int h = 0; h < MB / 2; ++h) {
          const double2 x = __ldg(xp + h);
          a1[2 * h] = fma(ae.x, x.x, a1[2 * h]);
          a1[2 * h + 1] = fma(ae.x, x.y, a1[2 * h + 1]);
          e1[2 * h] = fma(ae.y, x.x, e1[2 * h]);
          e1[2 * h + 1] = fma(ae.y, x.y, e1[2 * h + 1]);
        }
      } else {
        const double av = __ldcs(op.a.val + k);
#pragma unroll
        for (int h = 0; h < MB / 2; ++h) {
          const double2 x = __ldg(xp + h);
          a1[2 * h] = fma(av, x.x, a1[2 * h]);
          a1[2 * h + 1] = fma(av, x.y, a1[2 * h + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < MB; ++q) {
    a1[q] = sub_sum<V>(a1[q]);
    if (EM == E_SAMEPAT) e1[q] = sub_sum<V>(e1[q]);
  }
  if (row >= n) return;
#pragma unroll
  for (int q = 0; q < MB; ++q) {
    if (q % V != lane || q >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[q]];
    if (st.phase != PH_RUN) continue;
    double ex = e1[q];
    if (EM == E_IDENT) ex = xin[size_t(row) * MB + q];
    else if (EM == E_DIAG) ex = op.ediag[row] * xin[size_t(row) * MB + q];
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * ex + st.ca * a1[q]);
  }
}

// RHS-split variants: the 4 lanes of a row split the 8 right-hand sides (2
// each) and walk every nonzero of the row together, so one warp instruction
// gathers 8 rows x 64 contiguous bytes (two full sectors per nonzero instead
// of four half-used 16-byte pieces) and no cross-lane reduction is needed.
// (Loading each entry's column/value once per 4 lanes and passing them round
// with shuffles was measured slower: C3 chain 116 -> 167 ms, operator 106 ->
// 121 ms over 348 iterations.)
template <int EM, bool CHAIN>
__global__ void __launch_bounds__(256) k_spmv_il2(GmSolve* S, Group grp, CsrView f, OpView op,
                                                  const double* __restrict__ xin, double* __restrict__ xout) {
  if (!il_any_run(S, grp)) return;
  const int lane = threadIdx.x & 3;
  const int row = int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 2);
  const int n = CHAIN ? f.nrows : op.a.nrows;
  if (row >= n) return;
  const int* rp = CHAIN ? f.rowptr : op.a.rowptr;
  const int* ci = CHAIN ? f.colind : op.a.colind;
  const int b = rp[row], e = rp[row + 1];
  const double* xl = xin + 2 * lane;
  double a0 = 0.0, a1 = 0.0, e0 = 0.0, e1 = 0.0;
  int k = b;
#pragma unroll 4
  for (; k < e; ++k) {
    const int c = __ldg(ci + k);
    const double2 x = __ldg(reinterpret_cast<const double2*>(xl + size_t(c) * MB));
    if (CHAIN) {
      const double av = __ldg(f.val + k);
      a0 = fma(av, x.x, a0);
      a1 = fma(av, x.y, a1);
    } else if (EM == E_SAMEPAT) {
      const double2 ae = __ldg(op.ae + k);
      a0 = fma(ae.x, x.x, a0);
      a1 = fma(ae.x, x.y, a1);
      e0 = fma(ae.y, x.x, e0);
      e1 = fma(ae.y, x.y, e1);
    } else {
      const double av = __ldg(op.a.val + k);
      a0 = fma(av, x.x, a0);
      a1 = fma(av, x.y, a1);
    }
  }
  if (CHAIN) {
    reinterpret_cast<double2*>(xout + size_t(row) * MB)[lane] = make_double2(a0, a1);
    return;
  }
  const double2 xr = reinterpret_cast<const double2*>(xin + size_t(row) * MB)[lane];
  if (EM == E_IDENT) {
    e0 = xr.x;
    e1 = xr.y;
  } else if (EM == E_DIAG) {
    const double dd = op.ediag[row];
    e0 = dd * xr.x;
    e1 = dd * xr.y;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = 2 * lane + h;
    if (q >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[q]];
    if (st.phase != PH_RUN) continue;
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * (h ? e1 : e0) + st.ca * (h ? a1 : a0));
  }
}

// Row-binned k_spmv_il2 for irregular matrices (runtime.cuh row bins; C5's Zipf rows, where SELL-8 is
// declined for its padding): a row of class b gets L = 4, 4, 8, 16, 32 lanes -- L / 4 entry groups of the
// four right-hand-side-pair lanes -- so a 2 000-entry row is walked by a whole warp (8 entries per step)
// instead of by four lanes while the other 28 lanes of its warp idle. Partial sums of the entry groups are
// added by shuffles; blocks belong to one class each (offsets from the class counts, as on the host).
__host__ __device__ __forceinline__ int il2b_lanes(int b) { return b <= 1 ? 4 : 4 << (b - 1); }
__host__ __device__ __forceinline__ int il2b_blocks(const int* boff, int b) {
  return int((int64_t(boff[b + 1] - boff[b]) * il2b_lanes(b) + 255) / 256);
}
template <int EM, bool CHAIN>
__global__ void __launch_bounds__(256) k_spmv_il2b(GmSolve* S, Group grp, CsrView f, OpView op,
                                                   const double* __restrict__ xin, double* __restrict__ xout) {
  if (!il_any_run(S, grp)) return;
  const CsrView& m = CHAIN ? f : op.a;
  int b = 0, blk0 = 0;
  for (; b < NBIN; ++b) {
    const int nbk = il2b_blocks(m.boff, b);
    if (int(blockIdx.x) < blk0 + nbk) break;
    blk0 += nbk;
  }
  if (b == NBIN) return;
  const int L = il2b_lanes(b), G = L >> 2;
  const int t = (int(blockIdx.x) - blk0) * 256 + int(threadIdx.x);
  const int slot = t / L, l = t - slot * L;
  const int lane = l & 3, g = l >> 2;
  const bool ok = slot < m.boff[b + 1] - m.boff[b];
  const int row = ok ? m.brow[m.boff[b] + slot] : 0;
  const double* xl = xin + 2 * lane;
  double a0 = 0.0, a1 = 0.0, e0 = 0.0, e1 = 0.0;
  if (ok) {
    const int kb = m.rowptr[row], ke = m.rowptr[row + 1];
#pragma unroll 4
    for (int k = kb + g; k < ke; k += G) {
      const int c = __ldg(m.colind + k);
      const double2 x = __ldg(reinterpret_cast<const double2*>(xl + size_t(c) * MB));
      if (CHAIN) {
        const double av = __ldg(f.val + k);
        a0 = fma(av, x.x, a0);
        a1 = fma(av, x.y, a1);
      } else if (EM == E_SAMEPAT) {
        const double2 ae = __ldg(op.ae + k);
        a0 = fma(ae.x, x.x, a0);
        a1 = fma(ae.x, x.y, a1);
        e0 = fma(ae.y, x.x, e0);
        e1 = fma(ae.y, x.y, e1);
      } else {
        const double av = __ldg(op.a.val + k);
        a0 = fma(av, x.x, a0);
        a1 = fma(av, x.y, a1);
      }
    }
  }
  for (int o = 4; o < L; o <<= 1) {  // block-uniform: every lane of the warp takes part
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    if (!CHAIN && EM == E_SAMEPAT) {
      e0 += __shfl_xor_sync(0xffffffffu, e0, o);
      e1 += __shfl_xor_sync(0xffffffffu, e1, o);
    }
  }
  if (!ok || g != 0) return;
  if (CHAIN) {
    reinterpret_cast<double2*>(xout + size_t(row) * MB)[lane] = make_double2(a0, a1);
    return;
  }
  const double2 xr = reinterpret_cast<const double2*>(xin + size_t(row) * MB)[lane];
  if (EM == E_IDENT) {
    e0 = xr.x;
    e1 = xr.y;
  } else if (EM == E_DIAG) {
    const double dd = op.ediag[row];
    e0 = dd * xr.x;
    e1 = dd * xr.y;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = 2 * lane + h;
    if (q >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[q]];
    if (st.phase != PH_RUN) continue;
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * (h ? e1 : e0) + st.ca * (h ? a1 : a0));
  }
}

// SELL-8 variant of k_spmv_il2 (runtime.cuh Sell8): the same thread mapping (4
// lanes per row, lane q owns right-hand sides 2q, 2q + 1, 8 rows per warp), but
// step j's column index and value of the warp's 8 rows are 8 consecutive slots,
// so each is one request per warp instead of 8 scattered ones.
template <int EM, bool CHAIN>
__device__ __forceinline__ void sell8_rows(GmSolve* S, const Group& grp, const Sell8View& sv, const OpView& op,
                                           const double* __restrict__ xin, double* __restrict__ xout, int row) {
  const int lane = threadIdx.x & 3;
  if (row >= sv.nrows) return;
  const int e0 = __ldg(sv.sptr + (row >> 3)) + (row & 7);
  const int w = (__ldg(sv.sptr + (row >> 3) + 1) - __ldg(sv.sptr + (row >> 3))) >> 3;
  const double* xl = xin + 2 * lane;
  double a0 = 0.0, a1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll 8
  for (int j = 0; j < w; ++j) {
    const int e = e0 + 8 * j;
    const int c = __ldcs(sv.col + e);
    const double2 x = __ldg(reinterpret_cast<const double2*>(xl + size_t(c) * MB));
    if (!CHAIN && EM == E_SAMEPAT) {
      const double2 ae = __ldcs(sv.val2 + e);
      a0 = fma(ae.x, x.x, a0);
      a1 = fma(ae.x, x.y, a1);
      g0 = fma(ae.y, x.x, g0);
      g1 = fma(ae.y, x.y, g1);
    } else {
      const double av = __ldcs(sv.val + e);
      a0 = fma(av, x.x, a0);
      a1 = fma(av, x.y, a1);
    }
  }
  if (CHAIN) {
    reinterpret_cast<double2*>(xout + size_t(row) * MB)[lane] = make_double2(a0, a1);
    return;
  }
  if (EM == E_IDENT || EM == E_DIAG) {
    const double2 xr = reinterpret_cast<const double2*>(xin + size_t(row) * MB)[lane];
    const double dd = EM == E_DIAG ? op.ediag[row] : 1.0;
    g0 = dd * xr.x;
    g1 = dd * xr.y;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = 2 * lane + h;
    if (q >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[q]];
    if (st.phase != PH_RUN) continue;
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * (h ? g1 : g0) + st.ca * (h ? a1 : a0));
  }
}

template <int EM, bool CHAIN>
__global__ void __launch_bounds__(256) k_spmv_sell8(GmSolve* S, Group grp, Sell8View sv, OpView op,
                                                    const double* __restrict__ xin, double* __restrict__ xout) {
  if (!il_any_run(S, grp)) return;
  sell8_rows<EM, CHAIN>(S, grp, sv, op, xin, xout, int((blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 2));
}

// SM-affine persistent form: the 64-row blocks are split into one contiguous range per SM, and the CTAs
// resident on an SM take that SM's blocks in order (an atomic cursor per SM; an SM that runs dry steals from
// the others, so every block is done wherever the CTAs land). Rows that are neighbours in the mesh -- the
// +-1 line and +-1 plane entries of a stencil row -- are then gathered by the same SM within a short time,
// so the x-gather hits L1 instead of L2 (with the plain block order the co-resident CTAs of an SM are 148
// blocks apart and share nothing). ctr: [nsm + 1] zero on entry; the last CTA to finish zeroes it again.
template <int EM, bool CHAIN>
__global__ void __launch_bounds__(256) k_spmv_sell8p(GmSolve* S, Group grp, Sell8View sv, OpView op,
                                                     const double* __restrict__ xin, double* __restrict__ xout,
                                                     int* ctr, int nsm) {
  __shared__ int blk_s;
  if (il_any_run(S, grp)) {
    const int nblk = (sv.nrows + 63) / 64;
    const int per = (nblk + nsm - 1) / nsm;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int v = 0; v < nsm; ++v) {
      const int victim = int((smid + unsigned(v)) % unsigned(nsm));
      const int base = victim * per, lim = min(per, nblk - base);
      while (true) {
        __syncthreads();
        if (threadIdx.x == 0) blk_s = lim > 0 ? atomicAdd(ctr + victim, 1) : lim;
        __syncthreads();
        const int blk = blk_s;
        if (blk >= lim) break;
        sell8_rows<EM, CHAIN>(S, grp, sv, op, xin, xout, (base + blk) * 64 + int(threadIdx.x >> 2));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + nsm, 1) == int(gridDim.x) - 1) {
      for (int v = 0; v <= nsm; ++v) ctr[v] = 0;
      __threadfence();
    }
  }
}

// Halo-staged sliced-ELL variant (runtime.cuh HaloPattern): one CTA per block
// of HALO_R rows stages the block's halo of x (all MB right-hand sides, 64 B
// per column, the four 16-byte chunks XOR-swizzled by the row so the reads of
// 32 rows spread over the banks) into shared memory once with cp.async, then one thread per row walks its slice
// column-major: the matrix stream is a coalesced 2-byte local index + the value
// per entry and the x-gather never leaves the SM.
template <int EM, bool CHAIN>
__global__ void __launch_bounds__(4 * HALO_R) k_spmv_halo(GmSolve* S, Group grp, HaloView hv, OpView op,
                                                          const double* __restrict__ xin, double* __restrict__ xout) {
  if (!il_any_run(S, grp)) return;
  extern __shared__ double2 xs[];
  const int blk = blockIdx.x;
  const int h0 = hv.hoff[blk], L = hv.hoff[blk + 1] - h0;
  // stage the halo with asynchronous 16-byte copies (all in flight at once);
  // chunk h of halo row t lands in slot h ^ ((t >> 1) & 3) of the row so the
  // 16-byte reads of 8 rows x 4 chunks spread over the banks
  for (int i = threadIdx.x; i < 4 * L; i += 4 * HALO_R) {
    const int t = i >> 2, h = i & 3;
    const double* src = xin + size_t(__ldg(hv.halo + h0 + t)) * MB + 2 * h;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(xs + t * 4 + (h ^ ((t >> 1) & 3))));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // four threads per row, thread q of a row owns right-hand sides 2q, 2q + 1;
  // a warp covers 8 consecutive rows, so each entry's index and value loads
  // are 8 contiguous slots of the slice (one sector / one line per warp)
  const int q = threadIdx.x & 3;
  const int row = blk * HALO_R + (threadIdx.x >> 2);
  if (row >= hv.nrows) return;
  const int slice = row >> 5, lane = row & 31;
  const int e0 = __ldg(hv.sptr + slice), w = (__ldg(hv.sptr + slice + 1) - e0) >> 5;
  double a0 = 0.0, a1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll 8
  for (int j = 0; j < w; ++j) {
    const int e = e0 + j * 32 + lane;
    const int li = int(__ldcs(hv.lidx + e));
    const double2 x = xs[li * 4 + (q ^ ((li >> 1) & 3))];
    if (EM == E_SAMEPAT && !CHAIN) {
      const double2 v = __ldcs(hv.val2 + e);
      a0 = fma(v.x, x.x, a0);
      a1 = fma(v.x, x.y, a1);
      g0 = fma(v.y, x.x, g0);
      g1 = fma(v.y, x.y, g1);
    } else {
      const double v = __ldcs(hv.val + e);
      a0 = fma(v, x.x, a0);
      a1 = fma(v, x.y, a1);
    }
  }
  if (CHAIN) {
    reinterpret_cast<double2*>(xout + size_t(row) * MB)[q] = make_double2(a0, a1);
    return;
  }
  if (EM == E_IDENT || EM == E_DIAG) {
    const double dd = EM == E_DIAG ? op.ediag[row] : 1.0;
    const double2 xr = reinterpret_cast<const double2*>(xin + size_t(row) * MB)[q];
    g0 = dd * xr.x;
    g1 = dd * xr.y;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int qq = 2 * q + h;
    if (qq >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[qq]];
    if (st.phase != PH_RUN) continue;
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * (h ? g1 : g0) + st.ca * (h ? a1 : a0));
  }
}

// ---- dot: part[j][blk] = W_j . w (j <= k), part[k+1][blk] = ||w||^2 -------------
// which 0: w = W_{k+1} (projection h); which 1: w = W_{k+1} (probe d)
__global__ void __launch_bounds__(256) k_dot(GmSolve* S, int G) {
  GmSolve& st = S[blockIdx.y];
  if (st.phase != PH_RUN) return;
  extern __shared__ double sm[];
  double* wt = sm;              // DOT_TILE
  double* acc = sm + DOT_TILE;  // k + 2
  const int k = st.k, n = st.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = threadIdx.x; j <= k + 1; j += blockDim.x) acc[j] = 0.0;
  const double* w = st.V[k + 1];
  double wsq = 0.0;
  const int ntiles = (n + DOT_TILE - 1) / DOT_TILE;
  for (int t = blockIdx.x; t < ntiles; t += G) {
    const int r0 = t * DOT_TILE;
    const int rows = min(DOT_TILE, n - r0);
    __syncthreads();
    for (int i = threadIdx.x; i < DOT_TILE; i += blockDim.x) {
      const double v = i < rows ? w[vidx(r0 + i)] : 0.0;
      wt[i] = v;
      wsq = fma(v, v, wsq);
    }
    __syncthreads();
    for (int j = warp; j <= k; j += nw) {
      const double* vj = st.V[j];
      double p = 0.0;
#pragma unroll 4
      for (int i = lane; i < rows; i += 32) p = fma(vj[vidx(r0 + i)], wt[i], p);
      p = warp_sum(p);
      if (lane == 0) acc[j] += p;
    }
  }
  wsq = warp_sum(wsq);
  __syncthreads();
  if (lane == 0) wt[warp] = wsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += wt[i];
    acc[k + 1] = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= k + 1; j += blockDim.x) st.part[size_t(j) * G + blockIdx.x] = acc[j];
}

// ---- reduce partials: which 0 -> h (and w2_pre), 1 -> d (and w2_a) -------------
__global__ void k_reduce(GmSolve* S, int G, int which, int cnt) {
  GmSolve& st = S[blockIdx.y];
  if (st.phase != PH_RUN) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  const int k = st.k;
  if (j > k + 1) return;
  const double* p = st.part + size_t(j) * G;
  double s = 0.0;
  for (int i = lane; i < cnt; i += 32) s += p[i];
  s = warp_sum(s);
  if (lane != 0) return;
  if (j <= k) {
    (which == 0 ? st.h : st.d)[j] = st.scale[j] * s;
  } else {
    if (which == 0) st.w2_pre = s;
    else st.w2_a = s;
  }
}

// ---- update: w -= sum_j s_j c_j W_j  (mode 0: c = h; mode 1: c = d if reorth;
//      mode 2: u = sum_{j < asm_k} s_j y_j W_j for the assembly) -----------------
__global__ void __launch_bounds__(256) k_update(GmSolve* S, int G, int mode) {
  GmSolve& st = S[blockIdx.y];
  if (mode == 2 ? st.phase != PH_ASM : st.phase != PH_RUN) return;
  extern __shared__ double sm[];
  const int k = st.k;
  const int nj = mode == 2 ? st.asm_k : k + 1;
  double* coef = sm;                                              // nj
  const double** vp = reinterpret_cast<const double**>(sm + nj);  // nj
  __shared__ double red[8];
  __shared__ int do_it;
  if (mode == 1) {
    // Second pass only when ||d|| > 1e-10 ||w|| (and ||w|| > 0), gmres.cpp:108-119.
    if (threadIdx.x < 32) {
      double dn = 0.0;
      for (int j = threadIdx.x; j <= k; j += 32) dn = fma(st.d[j], st.d[j], dn);
      dn = warp_sum(dn);
      if (threadIdx.x == 0) do_it = (st.w2_a > 0.0 && dn > 1e-20 * st.w2_a) ? 1 : 0;
    }
    __syncthreads();
    if (!do_it) return;
  }
  const double* c = mode == 0 ? st.h : (mode == 1 ? st.d : st.y);
  for (int j = threadIdx.x; j < nj; j += blockDim.x) {
    coef[j] = st.scale[j] * c[j];
    vp[j] = st.V[j];
  }
  __syncthreads();
  const int n = st.n;
  double* w = mode == 2 ? st.ubuf : st.V[k + 1];
  double wsq = 0.0;
  const int ntiles = (n + UPD_TILE - 1) / UPD_TILE;
  for (int t = blockIdx.x; t < ntiles; t += G) {
    const int r = t * UPD_TILE + 2 * threadIdx.x;
    const int vr = vidx(r);               // basis vectors are chunk-major
    const int wr = mode == 2 ? r : vr;    // ubuf (assembly) is a flat vector
    if (r + 1 < n) {
      double2 a = mode == 2 ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(w + wr);
      const double sgn = mode == 2 ? 1.0 : -1.0;
      int j = 0;
      // eight vectors in flight per thread (the assembly's x = V y ran at 1.7 TB/s with four)
      for (; j + 8 <= nj; j += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const double2*>(vp[j + u] + vr);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a.x = fma(sgn * coef[j + u], v[u].x, a.x);
          a.y = fma(sgn * coef[j + u], v[u].y, a.y);
        }
      }
      for (; j + 4 <= nj; j += 4) {
        const double2 v0 = *reinterpret_cast<const double2*>(vp[j] + vr);
        const double2 v1 = *reinterpret_cast<const double2*>(vp[j + 1] + vr);
        const double2 v2 = *reinterpret_cast<const double2*>(vp[j + 2] + vr);
        const double2 v3 = *reinterpret_cast<const double2*>(vp[j + 3] + vr);
        a.x = fma(sgn * coef[j], v0.x, a.x);
        a.y = fma(sgn * coef[j], v0.y, a.y);
        a.x = fma(sgn * coef[j + 1], v1.x, a.x);
        a.y = fma(sgn * coef[j + 1], v1.y, a.y);
        a.x = fma(sgn * coef[j + 2], v2.x, a.x);
        a.y = fma(sgn * coef[j + 2], v2.y, a.y);
        a.x = fma(sgn * coef[j + 3], v3.x, a.x);
        a.y = fma(sgn * coef[j + 3], v3.y, a.y);
      }
      for (; j < nj; ++j) {
        const double2 v0 = *reinterpret_cast<const double2*>(vp[j] + vr);
        a.x = fma(sgn * coef[j], v0.x, a.x);
        a.y = fma(sgn * coef[j], v0.y, a.y);
      }
      *reinterpret_cast<double2*>(w + wr) = a;
      wsq = fma(a.x, a.x, fma(a.y, a.y, wsq));
    } else if (r < n) {
      double a = mode == 2 ? 0.0 : w[wr];
      const double sgn = mode == 2 ? 1.0 : -1.0;
      for (int j = 0; j < nj; ++j) a = fma(sgn * coef[j], vp[j][vr], a);
      w[wr] = a;
      wsq = fma(a, a, wsq);
    }
  }
  if (mode != 1) return;
  wsq = warp_sum(wsq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = wsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
    st.part[size_t(k + 1) * G + blockIdx.x] = s;
  }
}

constexpr int UP_MAXCOLS = 2048;  // largest k + 1 of the fused (clustered) Gram-Schmidt path

// ---- clustered, register-tiled Gram-Schmidt passes (the default path) -----------
// Measured on B200 (scripts/membench.cu): the read bandwidth of a
// many-vector tile walk is set by the contiguous bytes each CTA takes from one
// vector per tile -- 64 B: 2.3 TB/s, 128 B: 4.6 TB/s, 256 B: 6.1 TB/s, 512 B:
// 6.8 TB/s -- and by the bytes in flight per SM. So a tile of T rows x (k+1)
// basis vectors is split over a thread-block CLUSTER of CL CTAs by vectors:
// each CTA keeps T rows of only ~(k+1)/CL vectors in registers, which lets T
// stay at 64 rows (512 B per vector) up to k + 1 = 512 with the same register
// budget; the update's row sums are combined across the cluster through
// distributed shared memory (one cluster barrier per tile).
// Alternatives measured slower: shared-memory staging with cp.async, TMA 2-D
// boxes (32 rows x 8 vectors: 3.5 TB/s, op-rate bound), 1-D TMA per vector,
// an mbarrier producer/consumer ring, L2 prefetch, chunk-major basis layout.
//
// The kernel is persistent: all running solves' tiles form one list, split
// into contiguous ranges over the clusters, so every SM works whatever the
// number of solves in the batch. Partial results per cluster (slot) go to
// part[j][slot]; clusters that own no tile of a solve write zeros.
// UPDATE: w <- w - sum_j s_j h_j W_j, then part[j] = W_j . w_new (the measured
// second-pass probe, gmres.cpp:101-111) and part[k+1] = ||w_new||^2.
// !UPDATE: the projection, part[j] = W_j . w and part[k+1] = ||w||^2.
// Thread (rg, cg) owns rows {2 rg, 2 rg + 1} of local vectors cg, cg + CG, ...
// (GC_CPT = 8), loaded with 128-bit streaming loads; the loads of tile t+1 are
// issued before tile t is consumed (register double buffer).
constexpr int GC_THREADS = 512;
constexpr int GC_CPT = 8;
constexpr int GC_SMEM_DOUBLES = UP_MAXCOLS + UP_MAXCOLS + 2048 + 2 * 512 + 2 * 512 + 64;

// Row groups for c vectors per CTA: the largest power of two with
// (512 / RG) * GC_CPT >= c, capped at 256 (tile = 2 RG rows).
__host__ __device__ __forceinline__ int gc_rg(int c) {
  int rg = 256;
  while (rg > 2 && (GC_THREADS / rg) * GC_CPT < c) rg >>= 1;
  return rg;
}

template <int CL>
__device__ __forceinline__ void gc_cluster_sync() {
  if (CL > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
}

__device__ __forceinline__ double dsmem_ld(const double* p, int rank) {
  uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(p)), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

template <int RG, int CL, bool UPDATE>
__device__ __forceinline__ void gc_body(GmSolve& st, int G, int slot, int q, int ta, int tb, double* coef,
                                        const double** vp, double* red, double* wn, double* rowpart) {
  constexpr int CG = GC_THREADS / RG;
  constexpr int T = 2 * RG;
  constexpr int TPR = (GC_THREADS / T) < 32 ? (GC_THREADS / T) : 32;  // threads per row in the row sums
  constexpr int PPT = CG / TPR;
  constexpr int CGP = CG + 1;
  constexpr int RW = RG < 32 ? RG : 32;
  const int tid = threadIdx.x;
  const int rg = tid % RG, cg = tid / RG;
  const int my_row = tid / TPR, sub = tid % TPR;
  const int k = st.k, nj = k + 1, n = st.n;
  const int ld = (n + 31) & ~31;
  const int cpc = (nj + CL - 1) / CL;
  const int j0 = min(nj, q * cpc), ncol = min(nj, j0 + cpc) - j0;
  double* w = st.V[k + 1];
  __syncthreads();  // the previous segment is done with coef / vp / red
  for (int l = tid; l < ncol; l += GC_THREADS) {
    coef[l] = UPDATE ? st.scale[j0 + l] * st.h[j0 + l] : 0.0;
    vp[l] = st.V[j0 + l];
  }
  __syncthreads();
  const int ncol_me = ncol > cg ? min(GC_CPT, (ncol - cg + CG - 1) / CG) : 0;
  double dcol[GC_CPT];
#pragma unroll
  for (int c = 0; c < GC_CPT; ++c) dcol[c] = 0.0;
  double wsq = 0.0;
  auto load = [&](int t, double2* v, double2& w2, double& wp) {
    const int row = t * T + 2 * rg;
    const bool inb = t < tb && row < ld;
#pragma unroll
    for (int c = 0; c < GC_CPT; ++c)
      v[c] = (c < ncol_me && inb) ? __ldcs(reinterpret_cast<const double2*>(vp[cg + CG * c] + vidx(row)))
                                  : make_double2(0.0, 0.0);
    if (UPDATE) {
      const int rw = t * T + my_row;
      wp = (t < tb && sub == 0 && my_row < T && rw < n) ? w[vidx(rw)] : 0.0;
    } else {
      w2 = inb ? *reinterpret_cast<const double2*>(w + vidx(row)) : make_double2(0.0, 0.0);
    }
  };
  auto consume = [&](int t, const double2* v, double2 w2, double wpre, int par) {
    double w0, w1;
    if (UPDATE) {
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int c = 0; c < GC_CPT; ++c) {
        const double cfc = c < ncol_me ? coef[cg + CG * c] : 0.0;
        ax = fma(cfc, v[c].x, ax);
        ay = fma(cfc, v[c].y, ay);
      }
      red[(2 * rg) * CGP + cg] = ax;
      red[(2 * rg + 1) * CGP + cg] = ay;
      __syncthreads();
      double sacc = 0.0;
      if (my_row < T) {
#pragma unroll
        for (int u = 0; u < PPT; ++u) sacc += red[my_row * CGP + PPT * sub + u];
      }
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o, TPR);
      if (CL > 1) {
        double* rp = rowpart + par * 512;
        if (sub == 0 && my_row < T) rp[my_row] = sacc;
        gc_cluster_sync<CL>();
        if (sub == 0 && my_row < T) {
          double tot = 0.0;
#pragma unroll
          for (int r = 0; r < CL; ++r) tot += dsmem_ld(rp + my_row, r);
          sacc = tot;
        }
      }
      double* wb = wn + par * 512;
      if (sub == 0 && my_row < T) {
        const int rw = t * T + my_row;
        const bool valid = rw < n;
        const double wv = valid ? wpre - sacc : 0.0;
        if (valid && q == 0) w[vidx(rw)] = wv;
        wb[my_row] = wv;
        if (q == 0) wsq = fma(wv, wv, wsq);
      }
      __syncthreads();
      w0 = wb[2 * rg];
      w1 = wb[2 * rg + 1];
    } else {
      w0 = w2.x;
      w1 = w2.y;
      if (q == 0 && cg == 0) wsq = fma(w0, w0, fma(w1, w1, wsq));
    }
#pragma unroll
    for (int c = 0; c < GC_CPT; ++c) dcol[c] = fma(v[c].x, w0, fma(v[c].y, w1, dcol[c]));
  };
  double2 va[GC_CPT], vb[GC_CPT];
  double2 wa2, wb2;
  double wa = 0.0, wbv = 0.0;
  int t = ta, par = 0;
  load(t, va, wa2, wa);
  while (t < tb) {
    load(t + 1, vb, wb2, wbv);
    consume(t, va, wa2, wa, par);
    ++t;
    par ^= 1;
    if (t >= tb) break;
    load(t + 1, va, wa2, wa);
    consume(t, vb, wb2, wbv, par);
    ++t;
    par ^= 1;
  }
  // column sums over the RG row groups
  if (RG <= 32) {
#pragma unroll
    for (int c = 0; c < GC_CPT; ++c) {
      double x = dcol[c];
#pragma unroll
      for (int o = RW / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o, RW);
      if (rg == 0 && c < ncol_me) st.part[size_t(j0 + cg + CG * c) * G + slot] = x;
    }
  } else {
    constexpr int WPC = RG / 32;  // warps per column group
    __syncthreads();
#pragma unroll
    for (int c = 0; c < GC_CPT; ++c) {
      const double x = warp_sum(dcol[c]);
      if ((tid & 31) == 0) red[(c * CG + cg) * WPC + rg / 32] = x;
    }
    __syncthreads();
    if (tid < GC_CPT * CG) {
      const int c = tid / CG, g = tid % CG;
      double x = 0.0;
      for (int u = 0; u < WPC; ++u) x += red[(c * CG + g) * WPC + u];
      const int l = g + CG * c;
      if (l < ncol) st.part[size_t(j0 + l) * G + slot] = x;
    }
  }
  // ||w||^2 partial (rank 0 of the cluster)
  {
    const double x = warp_sum(wsq);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = x;
    __syncthreads();
    if (tid == 0 && q == 0) {
      double s = 0.0;
      for (int i = 0; i < GC_THREADS / 32; ++i) s += red[i];
      st.part[size_t(k + 1) * G + slot] = s;
    }
  }
}

__device__ __forceinline__ int gc_tiles(const GmSolve& st, int CL) {
  const int cpc = (st.k + 1 + CL - 1) / CL;
  const int T = 2 * gc_rg(cpc);
  return (st.n + T - 1) / T;
}

// Update + probe variants measured on C3 (k + 1 <= 335): three register buffers
// of 6 vectors instead of two of 8 (4.4 TB/s: memory-level parallelism is not
// what limits it); one barrier per tile with warp-shuffled row partials and 16
// broadcast loads per thread instead of the shared-memory row reduction (4.0
// TB/s: register spills); with clusters: a cluster barrier
// per tile for the row sums gives 3.3 / 2.7 TB/s for pairs / quads (the
// barrier's release waits for the in-flight loads of the next tile); a version
// that sends the row partials with st.async + mbarriers and defers the probe by
// one tile (tile parked in shared memory) reached 3.2 / 2.2 TB/s (shared-memory
// traffic, mbarrier spinning). Unclustered: 4.7 TB/s -- the default.

// Solves whose update pass runs in a TMA-staged kernel are skipped by the
// register-tiled update kernel.
constexpr int GT_MAXCOLS = 384;  // k_gs_tma: largest k + 1
constexpr int GX_NG = 12;        // k_gs_tmx: 32-vector groups per lane
constexpr int GX_MAXV = GX_NG * 32;  // k_gs_tmx: largest k + 2 (basis and w)
// Which update kernel owns a running solve this iteration. sel: bit 0 = k_gs_tma
// enabled, bit 1 = k_gs_tmx enabled; split: with both, k + 1 <= split goes to
// k_gs_tma (faster while k_gs_tmx's multi-chunk tiles are latency-bound, C3:
// k + 1 < ~190) and larger k to k_gs_tmx. 0 = the register-tiled kernel.
struct UpdSel {
  int sel, split;
  int proj;  // 1: the selector of the projection pass (bit 2: k_gs_tmx<true>)
  int low;   // update pass: k + 1 <= low stays on the register-tiled kernel
};
__device__ __forceinline__ int upd_owner(const GmSolve& st, UpdSel u) {
  const int nj = st.k + 1;
  if (nj <= u.low) return 0;
  if ((u.sel & 2) && st.tm != nullptr && nj + 1 <= GX_MAXV && (!(u.sel & 1) || nj > u.split)) return 2;
  if ((u.sel & 1) && nj <= GT_MAXCOLS) return 1;
  return 0;
}
__device__ __forceinline__ bool gt_handles(const GmSolve& st, UpdSel u) { return st.phase == PH_RUN && upd_owner(st, u) == 1; }
__device__ __forceinline__ bool gx_proj_owner(const GmSolve& st, UpdSel u) {
  return (u.sel & 4) && st.tm != nullptr && st.k + 2 <= GX_MAXV && st.k + 1 > u.split;
}
__device__ __forceinline__ bool gx_handles(const GmSolve& st, UpdSel u) {
  return st.phase == PH_RUN && (u.proj ? gx_proj_owner(st, u) : upd_owner(st, u) == 2);
}
// Delayed second pass (DCGS2-style, Swirydowicz et al. 2020): when the probe of
// iteration k asks for the second pass (gmres.cpp:108-119), the correction
// W_{k+1} -= sum_j d_j q_j is applied by iteration k + 1's projection pass
// (k_gs_tmx<true>, which reads the basis anyway), ||W_{k+1}||^2 is
// ||w||^2 - ||d||^2, and the projection of the next operator image on the
// corrected vector follows from the Arnoldi relation (k_dcgs_fix). Large
// corrections (||d||^2 > ||w||^2 / 4, where the Pythagorean norm loses digits)
// and iterations whose projection runs in the register-tiled kernel keep the
// immediate pass (k_reorth_p). ps: the projection selector.
__device__ __forceinline__ bool dcgs_lazy(const GmSolve& st, UpdSel ps, double dn) {
  const int k1 = st.k + 1;
  return st.dcgs && dn <= 0.25 * st.w2_a && k1 < st.max_iter && (ps.sel & 4) && st.tm != nullptr &&
         k1 + 2 <= GX_MAXV && k1 + 1 > ps.split;
}

template <int CL, bool UPDATE>
__global__ void __launch_bounds__(GC_THREADS, 1) k_gs_clu(GmSolve* S, int ns, int G, UpdSel skip) {
  extern __shared__ __align__(16) double smc[];
  double* coef = smc;
  const double** vp = reinterpret_cast<const double**>(smc + UP_MAXCOLS);
  double* red = smc + 2 * UP_MAXCOLS;
  double* wn = red + 2048;
  double* rowpart = wn + 2 * 512;
  const int q = int(blockIdx.x) % CL, slot = int(blockIdx.x) / CL, ncl = int(gridDim.x) / CL;
  long long total = 0;
  for (int s = 0; s < ns; ++s)
    if (S[s].phase == PH_RUN && (UPDATE ? upd_owner(S[s], skip) == 0 : !gx_proj_owner(S[s], skip))) total += gc_tiles(S[s], CL);
  const long long per = (total + ncl - 1) / ncl;
  const long long a = per * slot, b = min(total, a + per);
  long long off = 0;
  for (int s = 0; s < ns; ++s) {
    GmSolve& st = S[s];
    if (st.phase != PH_RUN || (UPDATE ? upd_owner(st, skip) != 0 : gx_proj_owner(st, skip))) continue;
    const int nt = gc_tiles(st, CL);
    const long long lo = a > off ? a : off, hi = b < off + nt ? b : off + nt;
    if (lo < hi) {
      const int ta = int(lo - off), tb = int(hi - off);
      const int cpc = (st.k + 1 + CL - 1) / CL;
      switch (gc_rg(cpc)) {
        case 256: gc_body<256, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 128: gc_body<128, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 64: gc_body<64, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 32: gc_body<32, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 16: gc_body<16, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 8: gc_body<8, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        case 4: gc_body<4, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
        default: gc_body<2, CL, UPDATE>(st, G, slot, q, ta, tb, coef, vp, red, wn, rowpart); break;
      }
    } else {
      // no tile of this solve here: zero partials for this CTA's vectors
      const int nj = st.k + 1, cpc = (nj + CL - 1) / CL;
      const int j0 = min(nj, q * cpc), j1 = min(nj, j0 + cpc);
      for (int j = j0 + int(threadIdx.x); j < j1; j += GC_THREADS) st.part[size_t(j) * G + slot] = 0.0;
      if (q == 0 && threadIdx.x == 0) st.part[size_t(nj) * G + slot] = 0.0;
    }
    off += nt;
  }
  gc_cluster_sync<CL>();  // peers may still read this CTA's row partials
}

// ---- measured second pass, persistent (gmres.cpp:108-119) ------------------------
// w <- w - sum_j s_j d_j W_j and ||w||^2 for the solves whose probe asked for it
// (||d|| > 1e-10 ||w||). The tiles (2048 rows, two per thread) of those solves
// form one list split over one 1024-thread CTA per SM, so the pass keeps every
// SM streaming (~128 KB of loads in flight) however many solves need it; the
// others skip. Slot b writes part[k+1][b] for every such solve (0 if it owned
// no tile), which k_finalize sums.
constexpr int RO_THREADS = 1024;
constexpr int RO_ROWS = 2 * RO_THREADS;

__global__ void __launch_bounds__(RO_THREADS, 1) k_reorth_p(GmSolve* S, int ns, int G, UpdSel ps) {
  extern __shared__ __align__(16) double smr[];
  double* coef = smr;
  const double** vp = reinterpret_cast<const double**>(smr + UP_MAXCOLS);
  double* red = smr + 2 * UP_MAXCOLS;               // 32
  int* need = reinterpret_cast<int*>(red + 32);     // ns flags
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int s = warp; s < ns; s += RO_THREADS / 32) {
    const GmSolve& st = S[s];
    int f = 0;
    if (st.phase == PH_RUN) {
      double dn = 0.0;
      for (int j = lane; j <= st.k; j += 32) dn = fma(st.d[j], st.d[j], dn);
      dn = warp_sum(dn);
      f = st.w2_a > 0.0 && dn > 1e-20 * st.w2_a && !dcgs_lazy(st, ps, dn);
    }
    if (lane == 0) need[s] = f;
  }
  __syncthreads();
  long long total = 0;
  for (int s = 0; s < ns; ++s)
    if (need[s]) total += (S[s].n + RO_ROWS - 1) / RO_ROWS;
  if (total == 0) return;
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long a = per * blockIdx.x, b = min(total, a + per);
  long long off = 0;
  for (int s = 0; s < ns; ++s) {
    if (!need[s]) continue;
    GmSolve& st = S[s];
    const int n = st.n, k = st.k, nj = k + 1;
    const int nt = (n + RO_ROWS - 1) / RO_ROWS;
    const long long lo = a > off ? a : off, hi = b < off + nt ? b : off + nt;
    off += nt;
    double wsq = 0.0;
    if (lo < hi) {
      __syncthreads();
      for (int j = tid; j < nj; j += RO_THREADS) {
        coef[j] = st.scale[j] * st.d[j];
        vp[j] = st.V[j];
      }
      __syncthreads();
      double* w = st.V[k + 1];
      for (long long t = lo - (off - nt); t < hi - (off - nt); ++t) {
        const int r = int(t) * RO_ROWS + 2 * tid;
        if (r + 1 < n) {
          const int vr = vidx(r);
          double2 acc = *reinterpret_cast<const double2*>(w + vr);
          int j = 0;
          for (; j + 8 <= nj; j += 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(vp[j + u] + vr));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              acc.x = fma(-coef[j + u], v[u].x, acc.x);
              acc.y = fma(-coef[j + u], v[u].y, acc.y);
            }
          }
          for (; j < nj; ++j) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(vp[j] + vr));
            acc.x = fma(-coef[j], v.x, acc.x);
            acc.y = fma(-coef[j], v.y, acc.y);
          }
          *reinterpret_cast<double2*>(w + vr) = acc;
          wsq = fma(acc.x, acc.x, fma(acc.y, acc.y, wsq));
        } else if (r < n) {
          const int vr = vidx(r);
          double x = w[vr];
          for (int j = 0; j < nj; ++j) x = fma(-coef[j], vp[j][vr], x);
          w[vr] = x;
          wsq = fma(x, x, wsq);
        }
      }
    }
    wsq = warp_sum(wsq);
    __syncthreads();
    if (lane == 0) red[warp] = wsq;
    __syncthreads();
    if (tid == 0) {
      double x = 0.0;
      for (int i = 0; i < RO_THREADS / 32; ++i) x += red[i];
      st.part[size_t(nj) * G + blockIdx.x] = x;
    }
  }
}

// ---- update + probe from TMA-staged tiles (default for k + 1 <= GT_MAXCOLS) ------
// Same contract as k_gs_clu<CL, true>: w <- w - sum_j s_j h_j W_j, part[j][slot]
// = W_j . w_new and part[k+1][slot] = ||w_new||^2. The register-tiled kernel has
// to hold a tile in registers across the barrier that completes its row sums,
// so its loads in flight stop at every tile (4.7 TB/s). Here the chunk-major
// basis is streamed with 1-D bulk copies (cp.async.bulk, one per 64-vector panel
// and chunk: m x 128 contiguous bytes) into a ring of NS shared-memory stages
// (one mbarrier each), so the copies of the next NS - 1 tiles stay in flight
// whatever the barriers do. Thread 0 refills a stage right after the tile's
// barrier: every warp has its elements in registers by then. (A dedicated
// producer warp makes 9 warps, i.e. 3 on one SM sub-partition, which caps the
// registers at 168 and spills.)
// Tile = TC consecutive 16-row chunks x all k + 2 vectors (w = W_{k+1} rides in
// the copy of the last panel). Warp w takes chunk cc = w / WPC and,
// within it, vectors j = i CPI + 2 (w % WPC) + (lane >> 4), row lane & 15: each
// element is read from shared memory once into a register, used for the row
// sum and, after the one barrier per tile that completes the row sums (row-sum
// buffers alternate between tiles), for the probe, whose per-vector
// partials stay in registers until the solve's last tile in this CTA.
constexpr int GT_CWARPS = 16;                      // warps
constexpr int GT_CONSUMERS = GT_CWARPS * 32;
constexpr int GT_THREADS = GT_CONSUMERS;
constexpr int GT_NI = 12;                          // vector slots per lane
static_assert(GT_MAXCOLS == GT_NI * 2 * GT_CWARPS, "k_gs_tma slots");
constexpr int GT_RING = 26 * 8192;                 // tile ring (bytes)
constexpr int GT_MAXST = 16;
constexpr int GT_SMEM = GT_RING + (2 * GT_CWARPS * 16 + GT_MAXCOLS + GT_CWARPS) * 8 + GT_MAXST * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ int gt_chunks(const GmSolve& st) { return ((st.n + 31) & ~31) / CHUNK; }
// SELL-8 SpMV with the matrix stream staged by TMA: a CTA owns 8 slices (64 rows), whose column indices and
// values are two contiguous runs of the SELL-8 arrays; one thread fetches both with bulk copies
// (cp.async.bulk) into shared memory and the CTA waits on the mbarrier. The stream then costs two DRAM-efficient
// requests per CTA instead of one 32-byte sector request per warp and step (k_spmv_sell8 is latency-bound on
// those: ncu long-scoreboard 45-67 %), never enters L1, and the only global loads left in the loop are the
// x-gathers; the loads of one CTA overlap the arithmetic of the others resident on the SM.
template <int EM, bool CHAIN>
__global__ void __launch_bounds__(256) k_spmv_sell8t(GmSolve* S, Group grp, Sell8View sv, OpView op,
                                                     const double* __restrict__ xin, double* __restrict__ xout) {
  extern __shared__ __align__(128) char s8sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int md[6];  // thread 0 reads the solve states for the CTA: any running, narrow mode and its slots
  constexpr bool PAIRV = !CHAIN && EM == E_SAMEPAT;
  constexpr int VB = PAIRV ? 16 : 8;
  const int nsl = (sv.nrows + 7) >> 3;
  const int s0 = int(blockIdx.x) * 8, s1 = min(nsl, s0 + 8);
  const int eb = __ldg(sv.sptr + s0), ee = __ldg(sv.sptr + s1);
  const int E = ee - eb;
  const int* cs = reinterpret_cast<const int*>(s8sm);
  const char* vs = s8sm + size_t(E) * 4;
  if (threadIdx.x < 32) il_mode_warp(S, grp, md);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (!md[5]) return;
  const bool NARROW = md[4] != 0;  // uniform over the grid
  const int nq0 = md[0], nq1 = md[1], nq2 = md[2], nq3 = md[3];
  if (threadIdx.x == 0 && E > 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    mbar_expect_tx(&bar, unsigned(E) * unsigned(4 + VB));
    bulk_g2s(s8sm, sv.col + eb, unsigned(E) * 4u, &bar, pol);
    if (PAIRV) bulk_g2s(s8sm + size_t(E) * 4, sv.val2 + eb, unsigned(E) * 16u, &bar, pol);
    else bulk_g2s(s8sm + size_t(E) * 4, sv.val + eb, unsigned(E) * 8u, &bar, pol);
  }
  const int lane = threadIdx.x & 3;
  const int ls = int(threadIdx.x >> 5);  // slice of this warp
  const int row = (s0 + ls) * 8 + int((threadIdx.x >> 2) & 7);
  int e0 = 0, w = 0;
  if (s0 + ls < s1) {
    const int a = __ldg(sv.sptr + s0 + ls);
    e0 = a - eb + (row & 7);
    w = (__ldg(sv.sptr + s0 + ls + 1) - a) >> 3;
  }
  const double* xl = xin + (NARROW ? lane : 2 * lane);
  if (E > 0) mbar_wait(&bar, 0);
  if (row >= sv.nrows) return;
  double a0 = 0.0, a1 = 0.0, g0 = 0.0, g1 = 0.0;
  if (NARROW) {
    // one right-hand side per lane: slot `lane` of x[row][4]
#pragma unroll 8
    for (int j = 0; j < w; ++j) {
      const int e = e0 + 8 * j;
      const int c = cs[e];
      const double x = __ldg(xl + size_t(c) * MBN);
      if (PAIRV) {
        const double2 ae = reinterpret_cast<const double2*>(vs)[e];
        a0 = fma(ae.x, x, a0);
        g0 = fma(ae.y, x, g0);
      } else {
        a0 = fma(reinterpret_cast<const double*>(vs)[e], x, a0);
      }
    }
    if (CHAIN) {
      xout[size_t(row) * MBN + lane] = a0;
      return;
    }
    const int q = lane == 0 ? nq0 : lane == 1 ? nq1 : lane == 2 ? nq2 : nq3;
    if (q < 0) return;
    if (EM == E_IDENT || EM == E_DIAG) g0 = (EM == E_DIAG ? op.ediag[row] : 1.0) * xin[size_t(row) * MBN + lane];
    GmSolve& st = S[grp.idx[q]];
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * g0 + st.ca * a0);
    return;
  }
#pragma unroll 8
  for (int j = 0; j < w; ++j) {
    const int e = e0 + 8 * j;
    const int c = cs[e];
    const double2 x = __ldg(reinterpret_cast<const double2*>(xl + size_t(c) * MB));
    if (PAIRV) {
      const double2 ae = reinterpret_cast<const double2*>(vs)[e];
      a0 = fma(ae.x, x.x, a0);
      a1 = fma(ae.x, x.y, a1);
      g0 = fma(ae.y, x.x, g0);
      g1 = fma(ae.y, x.y, g1);
    } else {
      const double av = reinterpret_cast<const double*>(vs)[e];
      a0 = fma(av, x.x, a0);
      a1 = fma(av, x.y, a1);
    }
  }
  if (CHAIN) {
    reinterpret_cast<double2*>(xout + size_t(row) * MB)[lane] = make_double2(a0, a1);
    return;
  }
  if (EM == E_IDENT || EM == E_DIAG) {
    const double2 xr = reinterpret_cast<const double2*>(xin + size_t(row) * MB)[lane];
    const double dd = EM == E_DIAG ? op.ediag[row] : 1.0;
    g0 = dd * xr.x;
    g1 = dd * xr.y;
  }
  if (2 * lane < grp.cnt && grp.half(2 * lane) == 1) {
    // a complex pair in columns 2 lane, 2 lane + 1: the 2 x 2 coupling of k_iter_op's pair form
    GmSolve& st = S[grp.idx[2 * lane]];
    if (st.phase != PH_RUN) return;
    const double sc = st.scale[st.k];
    double* w = st.V[st.k + 1];
    w[vidx(row)] = sc * (st.sre * g0 + st.ca * a0 + st.sim * g1);
    w[vidx(sv.nrows + row)] = sc * (-st.sim * g0 + st.sre * g1 + st.ca * a1);
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = 2 * lane + h;
    if (q >= grp.cnt) continue;
    GmSolve& st = S[grp.idx[q]];
    if (st.phase != PH_RUN) continue;
    st.V[st.k + 1][vidx(row)] = st.scale[st.k] * (st.sre * (h ? g1 : g0) + st.ca * (h ? a1 : a0));
  }
}


// Tile cursor over the handled solves: tiles [off, off + nt) belong to solve s.
struct GtCursor {
  int s = -1, nt = 0;
  long long off = 0;
  UpdSel us;
  __device__ __forceinline__ void seek(const GmSolve* S, int ns, int TC, long long g) {
    while (s < ns && (s < 0 || g >= off + nt)) {
      if (s >= 0) off += nt;
      ++s;
      while (s < ns && !gt_handles(S[s], us)) ++s;
      nt = s < ns ? (gt_chunks(S[s]) + TC - 1) / TC : 0;
    }
  }
};

// Stage layout: chunk cc of panel p at doubles (p TC + cc) 1024, [vector][16
// rows] inside (the last panel's chunks hold only its m vectors), so the
// offset of a warp's slot i is a compile-time constant plus a per-thread base.
// Producer state (thread 0): issues tile g into stage stg.
template <int TC>
struct GtProducer {
  GtCursor pc;
  const double* const* V = nullptr;
  int nv = 0, nchunks = 0;
  uint64_t pol = 0;
  // Called by all 32 lanes of warp 0: lane 0 arms the stage's mbarrier, then
  // lane l issues copy l (full panels first, then the last panel's chunks).
  __device__ __forceinline__ void issue(const GmSolve* S, int ns, long long g, int stg, int stage_bytes, char* ring,
                                        uint64_t* full, int lane) {
    if (pc.s < 0 || g >= pc.off + pc.nt) {
      pc.seek(S, ns, TC, g);
      const GmSolve& st = S[pc.s];
      V = st.V;
      nv = st.k + 2;  // basis vectors 0..k and w
      nchunks = gt_chunks(st);
    }
    const int c0 = int(g - pc.off) * TC;
    const int nch = min(TC, nchunks - c0);
    const int pf = nv >> 6, m = nv & 63;
    if (lane == 0) mbar_expect_tx(full + stg, unsigned(nch) * unsigned(nv) * 128u);
    __syncwarp();
    char* base = ring + size_t(stg) * size_t(stage_bytes);
    if (lane < pf) {
      bulk_g2s(base + size_t(lane) * TC * 8192, V[64 * lane] + size_t(c0) * 1024, unsigned(nch) * 8192u, full + stg,
               pol);
    } else if (m && lane < pf + nch) {
      const int q = lane - pf;
      bulk_g2s(base + size_t(pf * TC + q) * 8192, V[64 * pf] + size_t(c0 + q) * 1024, unsigned(m) * 128u, full + stg,
               pol);
    }
  }
};

template <int TC, int NI = GT_NI>
__device__ __forceinline__ void gt_body(GmSolve* S, int ns, int G, int stage_bytes, int NS, long long a, long long b,
                                        char* ring, uint64_t* full, double* red, double* red2, double* red3, UpdSel us) {
  constexpr int WPC = GT_CWARPS / TC;  // warps per chunk
  constexpr int CPI = 2 * WPC;         // vectors per slot step
  constexpr int SPP = 64 / CPI;        // slots per panel
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cc = warp / WPC, wq = warp % WPC, r = lane & 15, par = lane >> 4;
  const int slot = blockIdx.x;
  GtProducer<TC> prod;
  prod.pc.us = us;
  if (warp == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(prod.pol));
    for (long long g = a; g < b && g < a + NS; ++g) prod.issue(S, ns, g, int(g - a), stage_bytes, ring, full, lane);
  }
  GtCursor cu;
  cu.us = us;
  double coef[NI], acc[NI];
  double wsq = 0.0;
  double* w = nullptr;
  GmSolve* st = nullptr;
  int nj = 0, nchunks = 0, n = 0, woff = 0;
  const int tbase = cc * 1024 + (2 * wq + par) * 16 + r;
  long long seg_end = -1;
  int stg = 0;
  unsigned phase = 0;
  for (long long g = a; g < b; ++g) {
    const long long u = g - a;
    if (g >= seg_end) {  // first tile of a solve in this CTA
      cu.seek(S, ns, TC, g);
      seg_end = min(b, cu.off + cu.nt);
      st = S + cu.s;
      nj = st->k + 1;
      n = st->n;
      nchunks = gt_chunks(*st);
      w = st->V[nj];
      woff = ((nj >> 6) * TC + cc) * 1024 + (nj & 63) * 16 + r;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int j = i * CPI + 2 * wq + par;
        coef[i] = j < nj ? st->scale[j] * st->h[j] : 0.0;
        acc[i] = 0.0;
      }
      wsq = 0.0;
    }
    const int c0 = int(g - cu.off) * TC;
    const bool ccv = c0 + cc < nchunks;
    mbar_wait(full + stg, phase);
    const double* T = reinterpret_cast<const double*>(ring + size_t(stg) * size_t(stage_bytes)) + tbase;
    double v[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int j = i * CPI + 2 * wq + par;
      v[i] = (j < nj && ccv) ? T[(i / SPP) * TC * 1024 + (i % SPP) * CPI * 16] : 0.0;
    }
    const double wpre = ccv ? T[woff - tbase] : 0.0;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < NI; ++i) s4[i & 3] = fma(coef[i], v[i], s4[i & 3]);
    double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    double* rd = red + (u & 1) * (GT_CWARPS * 16);
    if (lane < 16) rd[warp * 16 + lane] = s;
    __syncthreads();  // row sums complete; every warp holds its part of the tile
    if (warp == 0 && g + NS < b) prod.issue(S, ns, g + NS, stg, stage_bytes, ring, full, lane);
    if (++stg == NS) {
      stg = 0;
      phase ^= 1u;
    }
    // row total over the chunk's WPC warps: each half-warp reads half of them
    double tot = 0.0;
    if (WPC >= 2) {
      constexpr int H = WPC / 2;
      double t2[2] = {0.0, 0.0};
#pragma unroll
      for (int q = 0; q < H; ++q) t2[q & 1] += rd[(cc * WPC + par * H + q) * 16 + r];
      tot = t2[0] + t2[1];
      tot += __shfl_xor_sync(0xffffffffu, tot, 16);
    } else {
      tot = rd[cc * 16 + r];
    }
    const double wn = wpre - tot;
    if (wq == 0 && lane < 16 && ccv && (c0 + cc) * CHUNK + r < n) {
      w[size_t(c0 + cc) * 1024 + r] = wn;
      wsq = fma(wn, wn, wsq);
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) acc[i] = fma(v[i], wn, acc[i]);
    if (g + 1 == seg_end) {  // flush this solve's partials
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        double x = acc[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        const int j = i * CPI + 2 * wq + par;
        if (r == 0 && j < nj) red2[cc * nj + j] = x;
      }
      const double x = warp_sum(wsq);
      if (lane == 0) red3[warp] = x;
      __syncthreads();
      for (int j = tid; j < nj; j += GT_CONSUMERS) {
        double y = 0.0;
        for (int q = 0; q < TC; ++q) y += red2[q * nj + j];
        st->part[size_t(j) * G + slot] = y;
      }
      if (tid == 0) {
        double y = 0.0;
        for (int q = 0; q < GT_CWARPS; ++q) y += red3[q];
        st->part[size_t(nj) * G + slot] = y;
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(GT_THREADS, 1) k_gs_tma(GmSolve* S, int ns, int G, UpdSel us) {
  extern __shared__ __align__(128) char smt[];
  char* ring = smt;
  double* red = reinterpret_cast<double*>(smt + GT_RING);  // [2][warps][16 rows]
  double* red2 = red + 2 * GT_CWARPS * 16;                  // [TC][k + 1]
  double* red3 = red2 + GT_MAXCOLS;                         // [warps]
  uint64_t* full = reinterpret_cast<uint64_t*>(red3 + GT_CWARPS);
  const int slot = blockIdx.x, nslots = gridDim.x;
  // Same tile geometry in every CTA: TC from the largest k + 1 handled.
  int njmax = 0;
  for (int s = 0; s < ns; ++s)
    if (gt_handles(S[s], us)) njmax = max(njmax, S[s].k + 1);
  if (njmax == 0) return;
  int TC = 1;
  while (TC < GT_CWARPS && njmax * 2 * TC <= GT_MAXCOLS) TC *= 2;
  const int stage_bytes = TC * ((njmax + 1 + 63) / 64) * 8192;
  const int NS = min(GT_MAXST, GT_RING / stage_bytes);
  long long total = 0;
  for (int s = 0; s < ns; ++s)
    if (gt_handles(S[s], us)) total += (gt_chunks(S[s]) + TC - 1) / TC;
  const long long per = (total + nslots - 1) / nslots;
  const long long a = min(total, per * slot), b = min(total, a + per);
  // zero partials of the handled solves with no tile here
  {
    long long off = 0;
    for (int s = 0; s < ns; ++s) {
      if (!gt_handles(S[s], us)) continue;
      const long long nt = (gt_chunks(S[s]) + TC - 1) / TC;
      if (!(a < off + nt && off < b)) {
        const int nj = S[s].k + 1;
        for (int j = int(threadIdx.x); j <= nj; j += GT_THREADS) S[s].part[size_t(j) * G + slot] = 0.0;
      }
      off += nt;
    }
  }
  if (a >= b) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // slot steps in use: ceil((k + 1) / CPI) in (6, 12]; a register tile of 8 / 10 / 12 slots avoids
  // issuing the empty ones (the same sizing as k_gs_tmx)
  const int used = (njmax + 2 * (GT_CWARPS / TC) - 1) / (2 * (GT_CWARPS / TC));
#define MPG_GT_CASE(T)                                                                              \
  case T:                                                                                           \
    if (used <= 8)                                                                                  \
      gt_body<T, 8>(S, ns, G, stage_bytes, NS, a, b, ring, full, red, red2, red3, us);              \
    else if (used <= 10)                                                                            \
      gt_body<T, 10>(S, ns, G, stage_bytes, NS, a, b, ring, full, red, red2, red3, us);             \
    else                                                                                            \
      gt_body<T>(S, ns, G, stage_bytes, NS, a, b, ring, full, red, red2, red3, us);                 \
    break;
  switch (TC) {
    MPG_GT_CASE(16)
    MPG_GT_CASE(8)
    MPG_GT_CASE(4)
    MPG_GT_CASE(2)
    default: gt_body<1>(S, ns, G, stage_bytes, NS, a, b, ring, full, red, red2, red3, us); break;
  }
#undef MPG_GT_CASE
}

// ---- update + probe without per-tile barriers (default for k + 2 <= GX_MAXV) -----
// Same contract as k_gs_clu<CL, true>. A producer warp streams tiles of TC
// chunks x all k + 2 vectors (w = W_{k+1} included) with 3-D tensor copies
// (cp.async.bulk.tensor) of each panel's [chunk][64 vectors][16 rows] block
// into a ring of NS stages (full/empty mbarriers). The copies use the 128-byte
// swizzle: the 16-byte unit holding rows (2q, 2q + 1) of vector j lands at unit
// q ^ (j & 7) of the vector's 128-byte line, so a warp can read one row pair of
// 32 consecutive vectors (lane l: vector 32 g + l) without bank conflicts.
// Consumer warp w owns row pair w of every chunk: its lanes hold 32-vector
// groups of the pair, the row sums are a warp butterfly (no CTA barrier), the
// probe partials stay in registers (vector 32 g + lane) until the solve's last
// tile here. The stage is released by one arrive per warp.
// (k_gs_tma, the barrier-per-tile version with 1-D bulk copies, is kept as an
// alternative: MPG_GS_UPD=tma.)
constexpr int GX_CWARPS = 8;                        // consumer warps (row pairs of a chunk)
constexpr int GX_THREADS = (GX_CWARPS + 1) * 32;    // + one producer warp
constexpr int GX_RING = 24 * 8192;                  // tile ring (bytes)
constexpr int GX_MAXST = 16;
constexpr int GX_SMEM = 1024 + GX_RING + (GX_CWARPS * GX_MAXV + GX_CWARPS) * 8 + 2 * GX_MAXST * 8;

__device__ __forceinline__ void tma3_g2s(uint32_t dst, const CUtensorMap* tm, int c1, int c2, uint32_t mbar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(dst),
      "l"(tm), "r"(0), "r"(c1), "r"(c2), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void consumers_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(GX_CWARPS * 32) : "memory"); }

struct GxCursor {
  int s = -1, nt = 0;
  long long off = 0;
  UpdSel us;
  __device__ __forceinline__ void seek(const GmSolve* S, int ns, int TC, long long g) {
    while (s < ns && (s < 0 || g >= off + nt)) {
      if (s >= 0) off += nt;
      ++s;
      while (s < ns && !gx_handles(S[s], us)) ++s;
      nt = s < ns ? (gt_chunks(S[s]) + TC - 1) / TC : 0;
    }
  }
};

__device__ __forceinline__ void gx_producer(GmSolve* S, int ns, int TC, int stage_bytes, int NS, long long a,
                                            long long b, uint32_t ring, uint64_t* full, uint64_t* empty, UpdSel us) {
  const int lane = threadIdx.x & 31;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  GxCursor pc;
  pc.us = us;
  const CUtensorMap* tm = nullptr;
  int nv = 0, nchunks = 0, stg = 0;
  unsigned eph = 0;  // parity of the empty barriers' current phase
  for (long long g = a; g < b; ++g) {
    if (g - a >= NS) mbar_wait(empty + stg, eph);
    if (pc.s < 0 || g >= pc.off + pc.nt) {
      pc.seek(S, ns, TC, g);
      const GmSolve& st = S[pc.s];
      tm = st.tm;
      nv = st.k + 2;
      nchunks = gt_chunks(st);
    }
    const int c0 = int(g - pc.off) * TC;
    const int nch = min(TC, nchunks - c0);
    const int pf = nv >> 6, mb = ((nv & 63) + 7) >> 3;  // full panels, 8-vector boxes of the last one
    const int per = pf + mb;
    if (lane == 0) mbar_expect_tx(full + stg, unsigned(nch) * unsigned(pf * 8192 + mb * 1024));
    __syncwarp();
    const uint32_t base = ring + uint32_t(stg) * uint32_t(stage_bytes);
    const uint32_t mbar = smem_u32(full + stg);
    for (int op = lane; op < nch * per; op += 32) {
      const int q = op / per, t = op - q * per;
      if (t < pf)
        tma3_g2s(base + uint32_t(t * TC + q) * 8192u, tm + 2 * t, 0, c0 + q, mbar, pol);
      else
        tma3_g2s(base + uint32_t(pf * TC) * 8192u + uint32_t(q * mb + t - pf) * 1024u, tm + 2 * pf + 1,
                 8 * (t - pf), c0 + q, mbar, pol);
    }
    if (++stg == NS) {
      stg = 0;
      if (g - a >= NS) eph ^= 1u;
    }
  }
}

// CF chunks of a tile are processed together (their load -> row sum -> butterfly
// chains interleave); each lane then holds NGC = GX_NG / CF groups per chunk, so
// CF = 1 serves k + 2 <= 384, CF = 2 <= 192, CF = 4 <= 96, CF = 8 <= 32.
template <int CF, bool PROJ, int NGT = GX_NG>
__device__ __forceinline__ void gx_consumer(GmSolve* S, int ns, int G, int TC, int stage_bytes, int NS, long long a,
                                            long long b, uint32_t ring, uint64_t* full, uint64_t* empty, double* red2,
                                            double* red3, UpdSel us) {
  constexpr int NGC = NGT / CF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int rp = warp;  // row pair
  const int slot = blockIdx.x;
  // byte offset of (vector 32 g + lane, row pair rp) inside a chunk of a stage
  const uint32_t loff = uint32_t(lane) * 128u + uint32_t((rp ^ (lane & 7)) << 4);
  GxCursor cu;
  cu.us = us;
  double coef[NGC], acc[NGC];
  double wsq = 0.0;
  double* w = nullptr;
  double* vk = nullptr;  // PROJ with pend: V[k] receives its delayed second-pass correction here
  bool pend = false;
  int nj = 0, nchunks = 0, n = 0, pf = 0, mb = 0;
  uint32_t woff = 0, vkoff = 0;
  long long seg_end = -1;
  int stg = 0;
  unsigned fph = 0;
  for (long long g = a; g < b; ++g) {
    if (g >= seg_end) {  // first tile of a solve in this CTA
      cu.seek(S, ns, TC, g);
      seg_end = min(b, cu.off + cu.nt);
      const GmSolve& st = S[cu.s];
      nj = st.k + 1;
      n = st.n;
      nchunks = gt_chunks(st);
      w = st.V[nj];
      pf = (nj + 1) >> 6;
      mb = (((nj + 1) & 63) + 7) >> 3;
      woff = uint32_t((rp ^ (nj & 7)) << 4) + uint32_t(nj & 63) * 128u;
      pend = PROJ && st.pend != 0;
      vk = st.V[nj - 1];
      vkoff = uint32_t((rp ^ ((nj - 1) & 7)) << 4) + uint32_t((nj - 1) & 63) * 128u;
#pragma unroll
      for (int i = 0; i < NGC; ++i) {
        const int j = 32 * i + lane;
        // the update coefficients, or (PROJ with pend) the correction coefficients of V[k]
        coef[i] = (!PROJ && j < nj) ? st.scale[j] * st.h[j] : (pend && j < nj - 1) ? st.scale[j] * st.dp[j] : 0.0;
        acc[i] = 0.0;
      }
      wsq = 0.0;
    }
    const int c0 = int(g - cu.off) * TC;
    mbar_wait(full + stg, fph);
    const uint32_t sbase = ring + uint32_t(stg) * uint32_t(stage_bytes);
    for (int cc0 = 0; cc0 < TC; cc0 += CF) {
      if (c0 + cc0 >= nchunks) break;
      // chunk cc of full panel p at (p TC + cc) 8 KB; of the last panel at
      // pf TC 8 KB + cc mb KB (its mb 8-vector boxes)
      double2 v[CF][NGC], wp[CF];
      double sx[CF], sy[CF];
#pragma unroll
      for (int f = 0; f < CF; ++f) {
        const int cc = cc0 + f;
        const bool ok = c0 + cc < nchunks;
        const uint32_t cb = sbase + uint32_t(cc) * 8192u;
        const uint32_t pb = sbase + uint32_t(pf * TC) * 8192u + uint32_t(cc * mb) * 1024u;
#pragma unroll
        for (int i = 0; i < NGC; ++i) {
          const uint32_t ad =
              ((i >> 1) < pf ? cb + uint32_t((i >> 1) * TC) * 8192u : pb) + uint32_t(i & 1) * 4096u + loff;
          v[f][i] = ok && 32 * i + lane < nj ? lds_f64x2(ad) : make_double2(0.0, 0.0);
        }
        wp[f] = ok ? lds_f64x2(((nj >> 6) < pf ? cb + uint32_t((nj >> 6) * TC) * 8192u : pb) + woff)
                   : make_double2(0.0, 0.0);
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int i = 0; i < ((PROJ && !pend) ? 0 : NGC); ++i) {
          if (i & 1) {
            x1 = fma(coef[i], v[f][i].x, x1);
            y1 = fma(coef[i], v[f][i].y, y1);
          } else {
            x0 = fma(coef[i], v[f][i].x, x0);
            y0 = fma(coef[i], v[f][i].y, y0);
          }
        }
        sx[f] = x0 + x1;
        sy[f] = y0 + y1;
      }
      if (!PROJ || pend) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int f = 0; f < CF; ++f) {
            sx[f] += __shfl_xor_sync(0xffffffffu, sx[f], o);
            sy[f] += __shfl_xor_sync(0xffffffffu, sy[f], o);
          }
      }
      if (PROJ && pend) {  // V[k] <- v~ - sum_{j<k} d_j q_j on this chunk's row pair
#pragma unroll
        for (int f = 0; f < CF; ++f) {
          const int cc = cc0 + f;
          if (lane == 0 && c0 + cc < nchunks) {
            const uint32_t cb = sbase + uint32_t(cc) * 8192u;
            const uint32_t pb = sbase + uint32_t(pf * TC) * 8192u + uint32_t(cc * mb) * 1024u;
            const double2 vkp =
                lds_f64x2((((nj - 1) >> 6) < pf ? cb + uint32_t(((nj - 1) >> 6) * TC) * 8192u : pb) + vkoff);
            const int row = (c0 + cc) * CHUNK + 2 * rp;
            double* dk = vk + size_t(c0 + cc) * 1024 + 2 * rp;
            if (row + 1 < n) *reinterpret_cast<double2*>(dk) = make_double2(vkp.x - sx[f], vkp.y - sy[f]);
            else if (row < n) dk[0] = vkp.x - sx[f];
          }
        }
      }
#pragma unroll
      for (int f = 0; f < CF; ++f) {
        const int cc = cc0 + f;
        // PROJ: w is only projected (sx holds the V[k] correction when pend)
        const double wn0 = PROJ ? wp[f].x : wp[f].x - sx[f], wn1 = PROJ ? wp[f].y : wp[f].y - sy[f];
        const int row = (c0 + cc) * CHUNK + 2 * rp;
        if (lane == 0 && c0 + cc < nchunks) {
          double* dst = w + size_t(c0 + cc) * 1024 + 2 * rp;
          if (row + 1 < n) {
            if (!PROJ) *reinterpret_cast<double2*>(dst) = make_double2(wn0, wn1);
            wsq = fma(wn0, wn0, fma(wn1, wn1, wsq));
          } else if (row < n) {
            if (!PROJ) dst[0] = wn0;
            wsq = fma(wn0, wn0, wsq);
          }
        }
#pragma unroll
        for (int i = 0; i < NGC; ++i) acc[i] = fma(v[f][i].x, wn0, fma(v[f][i].y, wn1, acc[i]));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stg);
    if (++stg == NS) {
      stg = 0;
      fph ^= 1u;
    }
    if (g + 1 == seg_end) {  // flush this solve's partials
      GmSolve& st = S[cu.s];
#pragma unroll
      for (int i = 0; i < NGC; ++i)
        if (32 * i + lane < nj) red2[warp * GX_MAXV + 32 * i + lane] = acc[i];
      if (lane == 0) red3[warp] = wsq;
      consumers_bar();
      for (int j = tid; j < nj; j += GX_CWARPS * 32) {
        double y = 0.0;
        for (int q = 0; q < GX_CWARPS; ++q) y += red2[q * GX_MAXV + j];
        st.part[size_t(j) * G + slot] = y;
      }
      if (tid == 0) {
        double y = 0.0;
        for (int q = 0; q < GX_CWARPS; ++q) y += red3[q];
        st.part[size_t(nj) * G + slot] = y;
      }
      consumers_bar();
    }
  }
}

// PROJ: the projection pass (part[j] = W_j . w, part[k+1] = ||w||^2, w unchanged).
template <bool PROJ>
__global__ void __launch_bounds__(GX_THREADS, 1) k_gs_tmx(GmSolve* S, int ns, int G, UpdSel us) {
  extern __shared__ __align__(1024) char smx[];
  const uint32_t raw = smem_u32(smx);
  const uint32_t ring = (raw + 1023u) & ~1023u;  // 128-byte swizzle needs 1024-byte aligned stages
  char* gen = smx + (ring - raw);
  double* red2 = reinterpret_cast<double*>(gen + GX_RING);  // [warps][GX_MAXV]
  double* red3 = red2 + GX_CWARPS * GX_MAXV;                 // [warps]
  uint64_t* full = reinterpret_cast<uint64_t*>(red3 + GX_CWARPS);
  uint64_t* empty = full + GX_MAXST;
  const int slot = blockIdx.x, nslots = gridDim.x;
  int nvmax = 0;
  for (int s = 0; s < ns; ++s)
    if (gx_handles(S[s], us)) nvmax = max(nvmax, S[s].k + 2);
  if (nvmax == 0) return;
  // tile = TC chunks of up to about 48 KB (at least 4 stages in the ring)
  const int chunk_bytes = (nvmax >> 6) * 8192 + (((nvmax & 63) + 7) >> 3) * 1024;
  const int CF = nvmax <= 32 ? 8 : nvmax <= 96 ? 4 : nvmax <= 192 ? 2 : 1;
  int TC = 1;
  while (TC < 16 && (TC < CF || 2 * TC * chunk_bytes <= 48 * 1024)) TC *= 2;
  const int stage_bytes = TC * chunk_bytes;
  const int NS = min(GX_MAXST, GX_RING / stage_bytes);
  long long total = 0;
  for (int s = 0; s < ns; ++s)
    if (gx_handles(S[s], us)) total += (gt_chunks(S[s]) + TC - 1) / TC;
  const long long per = (total + nslots - 1) / nslots;
  const long long a = min(total, per * slot), b = min(total, a + per);
  {
    long long off = 0;
    for (int s = 0; s < ns; ++s) {
      if (!gx_handles(S[s], us)) continue;
      const long long nt = (gt_chunks(S[s]) + TC - 1) / TC;
      if (!(a < off + nt && off < b)) {
        const int nj = S[s].k + 1;
        for (int j = int(threadIdx.x); j <= nj; j += GX_THREADS) S[s].part[size_t(j) * G + slot] = 0.0;
      }
      off += nt;
    }
  }
  if (a >= b) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, GX_CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= GX_CWARPS * 32)
    gx_producer(S, ns, TC, stage_bytes, NS, a, b, ring, full, empty, us);
  else
    switch (CF) {
      case 8: gx_consumer<8, PROJ>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us); break;
      case 4:
        if (nvmax <= 64)
          gx_consumer<4, PROJ, 8>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        else
          gx_consumer<4, PROJ>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        break;
      case 2:
        if (nvmax <= 128)  // groups past k + 2 cost issue slots, not bytes: size the register tile to k + 2
          gx_consumer<2, PROJ, 8>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        else if (nvmax <= 160)
          gx_consumer<2, PROJ, 10>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        else
          gx_consumer<2, PROJ>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        break;
      default:
        if (nvmax <= 256)
          gx_consumer<1, PROJ, 8>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        else if (nvmax <= 320)
          gx_consumer<1, PROJ, 10>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        else
          gx_consumer<1, PROJ>(S, ns, G, TC, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
        break;
    }
}

// ---- projection from a single-precision shadow of the basis -------------------------
// With the delayed second pass every iteration's new direction is measured against
// the basis by the update pass (the probe d = Q^T w_new, from the fp64 basis) and
// corrected by the next projection pass, so the first projection only has to remove
// most of the component in span(Q): its coefficients need a few digits, not sixteen.
// k_gs_tmxf therefore projects w on a float copy of the basis -- half the bytes of
// the pass -- while everything that defines the Arnoldi relation stays in fp64: the
// update pass subtracts the fp64 vectors, the probe is exact, H gets h~ + d, and the
// correction of V[k] (size ||d|| ~ 1e-7 ||w||) taken from the float copy is wrong by
// ~1e-7 ||d||, the same order as fp64 rounding.
// Shadow layout: panels [ld / 32][64][32] floats, i.e. 128 B per vector and chunk like
// the fp64 panels, so the tile geometry, the 128-byte swizzle and the ring of k_gs_tmx
// carry over with 32-row chunks: consumer warp q owns row quad q of every chunk (one
// float4 per vector). Columns 0..k-1 come from the shadow; w = W_{k+1} and V[k] (whose
// shadow does not exist yet: it may still await its correction) are staged in fp64 by
// 128-byte bulk copies. The kernel writes V[k]'s correction (fp64) and its shadow.
constexpr int FCHUNK = 32;
__host__ __device__ __forceinline__ int fidx(int r) { return (r / FCHUNK) * (PANEL * FCHUNK) + (r % FCHUNK); }
constexpr int GF_EXTRA = 512;  // per chunk and stage: 32 rows of w and of V[k] in fp64
constexpr int GF_SMEM = 1024 + GX_RING + (GX_CWARPS * GX_MAXV + 2 * GX_CWARPS) * 8 + 2 * GX_MAXST * 8;

__device__ __forceinline__ int gf_chunks(const GmSolve& st) { return ((st.n + 31) & ~31) / FCHUNK; }
// Boxes per chunk for nv shadow vectors: pf 64-vector boxes (8 KB) and mb 8-vector boxes (1 KB) of the last
// panel. Below 256 vectors an 8-vector box costs about twice its bytes (launch list, profiles/r02: k = 120,
// one panel + 7 small boxes, 2 315 us against 1 667 us for two full panels at k = 128), so from `mbfull`
// small boxes on the whole last panel is fetched instead; the vectors past nv are never read from the stage.
__device__ __forceinline__ void gf_split(int nv, int mbfull, int& pf, int& mb) {
  pf = nv >> 6;
  mb = ((nv & 63) + 7) >> 3;
  if (nv < 256 && mb >= mbfull) {
    ++pf;
    mb = 0;
  }
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, unsigned bytes, uint32_t mbar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

struct GfCursor {
  int s = -1, nt = 0;
  long long off = 0;
  UpdSel us;
  __device__ __forceinline__ void seek(const GmSolve* S, int ns, int TC, long long g) {
    while (s < ns && (s < 0 || g >= off + nt)) {
      if (s >= 0) off += nt;
      ++s;
      while (s < ns && !gx_handles(S[s], us)) ++s;
      nt = s < ns ? (gf_chunks(S[s]) + TC - 1) / TC : 0;
    }
  }
};

// Stage: the shadow tile as in k_gs_tmx (chunk cc of full panel p at (p TC + cc) 8 KB,
// the last panel's 8-vector boxes behind), then per chunk 512 B: w rows, V[k] rows.
__device__ __forceinline__ void gf_producer(GmSolve* S, int ns, int TC, int tile_bytes, int stage_bytes, int NS,
                                            long long a, long long b, uint32_t ring, uint64_t* full, uint64_t* empty,
                                            UpdSel us) {
  const int lane = threadIdx.x & 31;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  GfCursor pc;
  pc.us = us;
  const CUtensorMap* tm = nullptr;
  const double* w = nullptr;
  const double* vk = nullptr;
  int nv = 0, nchunks = 0, stg = 0;
  unsigned eph = 0;
  for (long long g = a; g < b; ++g) {
    if (g - a >= NS) mbar_wait(empty + stg, eph);
    if (pc.s < 0 || g >= pc.off + pc.nt) {
      pc.seek(S, ns, TC, g);
      const GmSolve& st = S[pc.s];
      tm = st.tmf;
      nv = st.k;  // shadow columns 0 .. k - 1
      nchunks = gf_chunks(st);
      w = st.V[st.k + 1];
      vk = st.V[st.k];
    }
    const int c0 = int(g - pc.off) * TC;
    const int nch = min(TC, nchunks - c0);
    int pf, mb;
    gf_split(nv, us.low & 0xff, pf, mb);
    const int per = pf + mb + 4;
    if (lane == 0) mbar_expect_tx(full + stg, unsigned(nch) * unsigned(pf * 8192 + mb * 1024 + GF_EXTRA));
    __syncwarp();
    const uint32_t base = ring + uint32_t(stg) * uint32_t(stage_bytes);
    const uint32_t mbar = smem_u32(full + stg);
    for (int op = lane; op < nch * per; op += 32) {
      const int q = op / per, t = op - q * per;
      if (t < pf) {
        tma3_g2s(base + uint32_t(t * TC + q) * 8192u, tm + 2 * t, 0, c0 + q, mbar, pol);
      } else if (t < pf + mb) {
        tma3_g2s(base + uint32_t(pf * TC) * 8192u + uint32_t(q * mb + t - pf) * 1024u, tm + 2 * pf + 1, 8 * (t - pf),
                 c0 + q, mbar, pol);
      } else {
        const int e = t - pf - mb;  // 0, 1: w; 2, 3: V[k] (the two 16-row fp64 chunks of this 32-row chunk)
        const double* src = (e < 2 ? w : vk) + size_t(2 * (c0 + q) + (e & 1)) * size_t(PANEL * CHUNK);
        bulk_g2s_a(base + uint32_t(tile_bytes) + uint32_t(q) * uint32_t(GF_EXTRA) + uint32_t(e) * 128u, src, 128u, mbar,
                   pol);
      }
    }
    if (++stg == NS) {
      stg = 0;
      if (g - a >= NS) eph ^= 1u;
    }
  }
}

// Arithmetic: the pass is issue-bound if every float is widened (4 F2F + 8 DFMA per lane and vector), so the
// four rows of a quad are contracted with single-precision FMAs -- the products already carry the shadow's
// 6e-8 rounding -- and only the 4-term partial is widened and accumulated in fp64; the correction's row sums
// (coefficients ~1e-7, a few digits needed) are summed in single precision across the warp.
// Packed single precision (FFMA2 / FMUL2 on sm_100a): two lanes of fp32 per instruction.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};\n" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;\n" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;\n" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void lds_b64x2(uint32_t a, uint64_t& lo, uint64_t& hi) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];\n" : "=l"(lo), "=l"(hi) : "r"(a));
}

template <int CF, int NGT>
__device__ __forceinline__ void gf_consumer(GmSolve* S, int ns, int G, int TC, int tile_bytes, int stage_bytes, int NS,
                                            long long a, long long b, uint32_t ring, uint64_t* full, uint64_t* empty,
                                            double* red2, double* red3, UpdSel us) {
  constexpr int NGC = NGT / CF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int rq = warp;  // row quad of a 32-row chunk
  const int slot = blockIdx.x;
  // the row of the quad whose sums end on this lane (transposed warp reduction below): lanes 8 u .. 8 u + 7 hold row u
  const int ur = lane >> 3;
  const bool tail_lane = (lane & 7) == 0;
  GfCursor cu;
  cu.us = us;
  // per vector group: the lane's float4 inside a stage (chunk 0) and its per-chunk stride; lanes past the
  // last vector read vector 0 (finite data) with a zero coefficient and never flush their sums, so the
  // chunk loop needs no per-load predicate or address select
  uint32_t goff[NGC], gstr[NGC];
  uint64_t coef2[NGC];
  double acc[NGC];
  double wsq = 0.0, acck = 0.0;  // on the tail lanes (0, 8, 16, 24: one row of the quad each)
  double* vk = nullptr;
  float* fk = nullptr;
  bool pend = false;
  int nj = 0, nv = 0, nchunks = 0, n = 0, pf = 0, mb = 0;
  long long seg_end = -1;
  int stg = 0;
  unsigned fph = 0;
  for (long long g = a; g < b; ++g) {
    if (g >= seg_end) {  // first tile of a solve in this CTA
      cu.seek(S, ns, TC, g);
      seg_end = min(b, cu.off + cu.nt);
      const GmSolve& st = S[cu.s];
      nj = st.k + 1;
      nv = nj - 1;
      n = st.n;
      nchunks = gf_chunks(st);
      gf_split(nv, us.low & 0xff, pf, mb);
      pend = st.pend != 0;
      vk = st.V[nj - 1];
      fk = st.F[nj - 1];
#pragma unroll
      for (int i = 0; i < NGC; ++i) {
        const int j = 32 * i + lane;
        const bool valid = j < nv;
        const int ii = valid ? i : 0, ll = valid ? lane : 0;
        const bool fullp = (ii >> 1) < pf;
        goff[i] = uint32_t(fullp ? (ii >> 1) * TC : pf * TC) * 8192u + uint32_t(ii & 1) * 4096u + uint32_t(ll) * 128u +
                  uint32_t((rq ^ (ll & 7)) << 4);
        gstr[i] = fullp ? 8192u : uint32_t(mb) * 1024u;
        const float cf = (pend && valid) ? float(st.scale[j] * st.dp[j]) : 0.f;  // the correction coefficients of V[k]
        coef2[i] = pk2(cf, cf);
        acc[i] = 0.0;
      }
      wsq = 0.0;
      acck = 0.0;
    }
    const int c0 = int(g - cu.off) * TC;
    mbar_wait(full + stg, fph);
    const uint32_t sbase = ring + uint32_t(stg) * uint32_t(stage_bytes);
    for (int cc0 = 0; cc0 < TC; cc0 += CF) {
      if (c0 + cc0 >= nchunks) break;
      uint64_t vlo[CF][NGC], vhi[CF][NGC];
      uint64_t w01[CF], w23[CF];
      float sx[CF];  // after the reduction: the correction's sum for row ur of the quad
#pragma unroll
      for (int f = 0; f < CF; ++f) {
        const int cc = cc0 + f;
        const bool ok = f == 0 || c0 + cc < nchunks;  // (uniform) a tile's last chunk pair may be half empty
        const uint32_t xb = sbase + uint32_t(tile_bytes) + uint32_t(cc) * uint32_t(GF_EXTRA) + uint32_t(rq) * 32u;
        if (ok) {
#pragma unroll
          for (int i = 0; i < NGC; ++i) lds_b64x2(sbase + goff[i] + uint32_t(cc) * gstr[i], vlo[f][i], vhi[f][i]);
          const double2 wlo = lds_f64x2(xb);
          const double2 whi = lds_f64x2(xb + 16u);
          w01[f] = pk2(float(wlo.x), float(wlo.y));
          w23[f] = pk2(float(whi.x), float(whi.y));
        } else {
#pragma unroll
          for (int i = 0; i < NGC; ++i) vlo[f][i] = vhi[f][i] = 0ull;
          w01[f] = w23[f] = 0ull;
        }
        sx[f] = 0.f;
        if (pend) {
          uint64_t x01 = 0ull, x23 = 0ull;
#pragma unroll
          for (int i = 0; i < NGC; ++i) {
            x01 = fma2(coef2[i], vlo[f][i], x01);
            x23 = fma2(coef2[i], vhi[f][i], x23);
          }
          // transposed reduction: 6 shuffles instead of 20; row u's sum ends on lanes 8 u .. 8 u + 7
          float x0, x1, x2, x3;
          upk2(x01, x0, x1);
          upk2(x23, x2, x3);
          const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0;
          const float s0 = hi16 ? x0 : x2, s1 = hi16 ? x1 : x3;
          const float y0 = (hi16 ? x2 : x0) + __shfl_xor_sync(0xffffffffu, s0, 16);
          const float y1 = (hi16 ? x3 : x1) + __shfl_xor_sync(0xffffffffu, s1, 16);
          float z = (hi8 ? y1 : y0) + __shfl_xor_sync(0xffffffffu, hi8 ? y0 : y1, 8);
          z += __shfl_xor_sync(0xffffffffu, z, 4);
          z += __shfl_xor_sync(0xffffffffu, z, 2);
          z += __shfl_xor_sync(0xffffffffu, z, 1);
          sx[f] = z;
        }
      }
#pragma unroll
      for (int f = 0; f < CF; ++f) {
        const int cc = cc0 + f;
        if (tail_lane && c0 + cc < nchunks) {
          // row ur of the quad: V[k] staged (uncorrected) for h'_k, corrected to global, shadow written
          const uint32_t xb = sbase + uint32_t(tile_bytes) + uint32_t(cc) * uint32_t(GF_EXTRA) + uint32_t(rq) * 32u +
                              uint32_t(ur) * 8u;
          double wv, yv;
          asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(wv) : "r"(xb));
          asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(yv) : "r"(xb + 256u));
          acck = fma(yv, wv, acck);
          wsq = fma(wv, wv, wsq);
          const double uv = yv - double(sx[f]);
          const int row = (c0 + cc) * FCHUNK + 4 * rq + ur;
          if (row < n) {
            if (pend) vk[vidx(row)] = uv;
            fk[fidx(row)] = float(uv);
          }
        }
#pragma unroll
        for (int i = 0; i < NGC; ++i) {
          const uint64_t p2 = fma2(vhi[f][i], w23[f], mul2(vlo[f][i], w01[f]));
          float pa, pb;
          upk2(p2, pa, pb);
          acc[i] += double(pa + pb);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stg);
    if (++stg == NS) {
      stg = 0;
      fph ^= 1u;
    }
    if (g + 1 == seg_end) {  // flush this solve's partials
      GmSolve& st = S[cu.s];
#pragma unroll
      for (int i = 0; i < NGC; ++i)
        if (32 * i + lane < nv) red2[warp * GX_MAXV + 32 * i + lane] = acc[i];
      const double wsum = warp_sum(wsq), ksum = warp_sum(acck);
      if (lane == 0) {
        red3[warp] = wsum;
        red3[GX_CWARPS + warp] = ksum;
      }
      consumers_bar();
      for (int j = tid; j < nv; j += GX_CWARPS * 32) {
        double y = 0.0;
        for (int q = 0; q < GX_CWARPS; ++q) y += red2[q * GX_MAXV + j];
        st.part[size_t(j) * G + slot] = y;
      }
      if (tid < 2) {
        double y = 0.0;
        for (int q = 0; q < GX_CWARPS; ++q) y += red3[tid * GX_CWARPS + q];
        st.part[size_t(tid == 0 ? nj : nv) * G + slot] = y;
      }
      consumers_bar();
    }
  }
}

__global__ void __launch_bounds__(GX_THREADS, 1) k_gs_tmxf(GmSolve* S, int ns, int G, UpdSel us) {
  extern __shared__ __align__(1024) char smx[];
  const uint32_t raw = smem_u32(smx);
  const uint32_t ring = (raw + 1023u) & ~1023u;
  char* gen = smx + (ring - raw);
  double* red2 = reinterpret_cast<double*>(gen + GX_RING);  // [warps][GX_MAXV]
  double* red3 = red2 + GX_CWARPS * GX_MAXV;                 // [2][warps]
  uint64_t* full = reinterpret_cast<uint64_t*>(red3 + 2 * GX_CWARPS);
  uint64_t* empty = full + GX_MAXST;
  const int slot = blockIdx.x, nslots = gridDim.x;
  int nvmax = 0;
  for (int s = 0; s < ns; ++s)
    if (gx_handles(S[s], us)) nvmax = max(nvmax, S[s].k);
  bool any = false;
  for (int s = 0; s < ns; ++s) any = any || gx_handles(S[s], us);
  if (!any) return;
  int pfm, mbm;
  gf_split(nvmax, us.low & 0xff, pfm, mbm);
  const int chunk_bytes = pfm * 8192 + mbm * 1024;
  const int CF = nvmax <= (us.low >> 8) ? 2 : 1;  // two chunks per consumer step up to this many vectors
  int TC = 1;
  while (TC < 16 && (TC < CF || 2 * TC * (chunk_bytes + GF_EXTRA) <= 48 * 1024)) TC *= 2;
  const int tile_bytes = TC * chunk_bytes;
  const int stage_bytes = (tile_bytes + TC * GF_EXTRA + 1023) & ~1023;
  const int NS = min(GX_MAXST, GX_RING / stage_bytes);
  long long total = 0;
  for (int s = 0; s < ns; ++s)
    if (gx_handles(S[s], us)) total += (gf_chunks(S[s]) + TC - 1) / TC;
  const long long per = (total + nslots - 1) / nslots;
  const long long a = min(total, per * slot), b = min(total, a + per);
  {
    long long off = 0;
    for (int s = 0; s < ns; ++s) {
      if (!gx_handles(S[s], us)) continue;
      const long long nt = (gf_chunks(S[s]) + TC - 1) / TC;
      if (!(a < off + nt && off < b)) {
        const int nj = S[s].k + 1;
        for (int j = int(threadIdx.x); j <= nj; j += GX_THREADS) S[s].part[size_t(j) * G + slot] = 0.0;
      }
      off += nt;
    }
  }
  if (a >= b) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, GX_CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= GX_CWARPS * 32)
    gf_producer(S, ns, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, us);
  else if (CF == 2) {
    if (nvmax <= 128)
      gf_consumer<2, 8>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else if (nvmax <= 160)
      gf_consumer<2, 10>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else if (nvmax <= 192)
      gf_consumer<2, 12>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else if (nvmax <= 224)
      gf_consumer<2, 14>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else
      gf_consumer<2, 16>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
  } else {
    if (nvmax <= 256)
      gf_consumer<1, 8>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else if (nvmax <= 320)
      gf_consumer<1, 10>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
    else
      gf_consumer<1, 12>(S, ns, G, TC, tile_bytes, stage_bytes, NS, a, b, ring, full, empty, red2, red3, us);
  }
}

// Shadow of V[k] for the solves whose projection runs in a fp64 kernel this iteration
// (V[k] is final there: no correction is pending); k_gs_tmxf writes the others'.
__global__ void __launch_bounds__(256) k_shadow(GmSolve* S, UpdSel ps) {
  GmSolve& st = S[blockIdx.y];
  if (st.phase != PH_RUN || st.F == nullptr || gx_proj_owner(st, ps)) return;
  const double* v = st.V[st.k];
  float* f = st.F[st.k];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < st.n; r += gridDim.x * blockDim.x) f[fidx(r)] = float(v[vidx(r)]);
}

// ---- norm partials of the residual buffer ----------------------------------------
__global__ void __launch_bounds__(256) k_rnorm(GmSolve* S, int G) {
  GmSolve& st = S[blockIdx.y];
  if (st.phase != PH_ASM) return;
  __shared__ double red[8];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += G * blockDim.x) s = fma(st.rbuf[i], st.rbuf[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += red[i];
    st.part[blockIdx.x] = t;
  }
}

__device__ void enter_finish(GmSolve& st, int kk, bool guess) {
  if (kk > 0) {
    st.phase = PH_ASM;
    st.asm_kind = ASM_FINISH;
    st.asm_k = kk;
    st.guess = guess;
  } else {
    st.final_residual = st.bnorm;
    st.converged = guess && st.bnorm <= st.target;
    st.xsel = -1;  // x = 0
    st.phase = PH_DONE;
  }
}

__device__ void continue_iter(GmSolve& st) {
  st.scale[st.k + 1] = 1.0 / st.wn_cur;
  st.k += 1;
  if (st.k >= st.max_iter) enter_finish(st, st.iterations, st.estimate <= st.target);
}

// ---- delayed second pass: coefficients of this iteration (DCGS2) ------------------
// With pend, the projection pass corrected V[k] (v~ -> u = v~ - sum_{j<k} d_j q_j)
// while projecting the operator image w' = A P (s_k v~) = A P q_k + s_k sum_j d_j A P q_j
// on the staged v~: h'_j = q_j . w' (j < k), h'_k = s_k v~ . w'. Then
//   c_k = q_k . w' = h'_k - s_k sum_{j<k} d_j h'_j, c_j = h'_j,
//   Hessenberg column hg_i = c_i - s_k (H~ d)_i (Arnoldi: A P q_j = sum_i H~_ij q_i),
// and the update pass removes sum_j c_j q_j from w' (h[k] = c_k): the same new
// direction as for the true image, whose projection is hg. Without a pending
// correction hg = h.
__global__ void __launch_bounds__(256) k_dcgs_fix(GmSolve* S) {
  static_assert(UP_MAXCOLS <= 8 * 256, "k_dcgs_fix rows per thread");
  GmSolve& st = S[blockIdx.x];
  if (st.phase != PH_RUN || !st.dcgs) return;
  const int k = st.k;
  double* h = st.h;
  if (!st.pend) {
    for (int j = threadIdx.x; j <= k; j += blockDim.x) st.hg[j] = h[j];
    return;
  }
  __shared__ double red[8];
  __shared__ double ck_s;
  const double* dp = st.dp;
  double t = 0.0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) t = fma(dp[j], h[j], t);
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  const double sk = st.scale[k];
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) x += red[i];
    ck_s = h[k] - sk * x;
  }
  __syncthreads();
  const double ck = ck_s;
  // (H~ d)_i = sum_{j < k, j + 1 >= i} H~_ij d_j, column by column so the reads of
  // each stored column are coalesced; a thread keeps rows tid, tid + 256, ...
  constexpr int RPT = 8;  // rows per thread: k + 1 <= 2048 (UP_MAXCOLS)
  double hd[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) hd[u] = 0.0;
  // (the loop is a chain of L2 round trips unless several columns are in flight: 8 per step,
  // and only the row slots a basis of k + 1 vectors reaches)
  const int nu = min(RPT, (k + 256) / 256);
  int j = 0;
  for (; j + 8 <= k; j += 8) {
    double cv[8][RPT];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double* col = st.Hu + hoff2(j + c);
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = threadIdx.x + u * 256;
        cv[c][u] = (u < nu && i <= j + c + 1) ? col[i] : 0.0;
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double dj = dp[j + c];
#pragma unroll
      for (int u = 0; u < RPT; ++u) hd[u] = fma(cv[c][u], dj, hd[u]);
    }
  }
  for (; j < k; ++j) {
    const double dj = dp[j];
    const double* col = st.Hu + hoff2(j);
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = threadIdx.x + u * 256;
      if (i <= j + 1) hd[u] = fma(col[i], dj, hd[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int i = threadIdx.x + u * 256;
    if (i <= k) st.hg[i] = (i < k ? h[i] : ck) - sk * hd[u];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    h[k] = ck;
    st.pend = 0;
  }
}

// ---- finalize the iteration: reorth bookkeeping, Givens, decisions ----------------
__global__ void k_finalize(GmSolve* S, int G, int cnt2, UpdSel ps) {
  GmSolve& st = S[blockIdx.x];
  if (st.phase != PH_RUN) return;
  const int lane = threadIdx.x;
  const int k = st.k;
  double* h = st.dcgs ? st.hg : st.h;  // the Hessenberg column (k_dcgs_fix) / the update coefficients
  double dn = 0.0;
  for (int j = lane; j <= k; j += 32) dn = fma(st.d[j], st.d[j], dn);
  dn = warp_sum(dn);
  const bool reorth = st.w2_a > 0.0 && dn > 1e-20 * st.w2_a;
  const bool lazy = reorth && dcgs_lazy(st, ps, dn);
  double w2 = st.w2_a;
  if (lazy) {
    w2 = st.w2_a - dn;  // ||w - Q d||^2 with d = Q^T w
    for (int j = lane; j <= k; j += 32) {
      h[j] += st.d[j];
      st.dp[j] = st.d[j];
    }
  } else if (reorth) {
    double s = 0.0;
    for (int i = lane; i < cnt2; i += 32) s += st.part[size_t(k + 1) * G + i];
    w2 = warp_sum(s);
    for (int j = lane; j <= k; j += 32) h[j] += st.d[j];
  }
  __syncwarp();
  if (lane != 0) return;
  st.pend = lazy ? 1 : 0;
  st.w2_b = w2;
  st.reorth_count += reorth;
  const double wnorm = sqrt(w2);
  const double wnorm_pre = sqrt(st.w2_pre);
  const bool invariant = wnorm <= 1e-14 * fmax(wnorm_pre, 1e-300);
  h[k + 1] = invariant ? 0.0 : wnorm;
  if (st.dcgs) {  // unrotated column k for the next corrections' H d products
    double* hu = st.Hu + hoff2(k);
    for (int i = 0; i <= k + 1; ++i) hu[i] = h[i];
  }
  // previous rotations (gmres.cpp:125-134); the rotated entry is carried in a
  // register so only the independent loads sit on the loop
  double hi = h[0];
#pragma unroll 4
  for (int i = 0; i < k; ++i) {
    const double c = st.cs[i], s = st.sn[i], hn = h[i + 1];
    h[i] = c * hi + s * hn;
    hi = -s * hi + c * hn;
  }
  h[k] = hi;
  const double diag = h[k], sub = h[k + 1];
  if (diag == 0.0 && sub == 0.0) {
    st.breakdown = 1;
    st.iterations = k;
    enter_finish(st, k, st.estimate <= st.target);
    return;
  }
  const double denom = hypot(diag, sub);
  const double c = diag / denom, s = sub / denom;
  st.cs[k] = c;
  st.sn[k] = s;
  h[k] = denom;
  double* Hk = st.H + hoff(k);
  for (int i = 0; i <= k; ++i) Hk[i] = h[i];
  st.g[k + 1] = -s * st.g[k];
  st.g[k] = c * st.g[k];
  st.estimate = fabs(st.g[k + 1]);
  st.iterations = k + 1;
  if (st.record) st.hist[k + 1] = st.estimate;
  st.wn_cur = wnorm;
  if (invariant) {
    st.breakdown = st.estimate > st.target;
    enter_finish(st, k + 1, st.estimate <= st.target);
    return;
  }
  if (st.estimate <= st.recheck_at) {
    st.phase = PH_ASM;
    st.asm_kind = ASM_RECHECK;
    st.asm_k = k + 1;
    return;
  }
  continue_iter(st);
}

// ---- assembly: y = R^{-1} g (column-oriented back substitution) ----------------------
__global__ void __launch_bounds__(256) k_backsub(GmSolve* S) {
  GmSolve& st = S[blockIdx.x];
  if (st.phase != PH_ASM) return;
  extern __shared__ double ys[];
  const int kk = st.asm_k;
  for (int i = threadIdx.x; i < kk; i += blockDim.x) ys[i] = st.g[i];
  __syncthreads();
  for (int i = kk - 1; i >= 0; --i) {
    const double* Hi = st.H + hoff(i);
    const double yi = ys[i] / Hi[i];
    __syncthreads();
    for (int t = threadIdx.x; t < i; t += blockDim.x) ys[t] = fma(-Hi[t], yi, ys[t]);
    if (threadIdx.x == 0) ys[i] = yi;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < kk; i += blockDim.x) st.y[i] = ys[i];
}

// ---- assembly post: recheck / finish decisions ----------------------------------------
__global__ void k_post(GmSolve* S, int G) {
  GmSolve& st = S[blockIdx.x];
  if (st.phase != PH_ASM) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < G; i += 32) s += st.part[i];
  s = warp_sum(s);
  if (threadIdx.x != 0) return;
  const double tr = sqrt(s);
  st.xsel = st.stages ? 1 + ((st.stages - 1) & 1) : 0;
  if (st.asm_kind == ASM_RECHECK) {
    if (tr <= st.target) {
      st.final_residual = tr;
      st.converged = 1;
      st.phase = PH_DONE;
      return;
    }
    st.recheck_at *= 0.25;
    st.phase = PH_RUN;
    continue_iter(st);
  } else {
    st.final_residual = tr;
    st.converged = st.guess && tr <= st.target;
    st.phase = PH_DONE;
  }
}

__global__ void k_init(GmSolve* S, int G) {
  // bnorm from the rbuf partials written by k_rnorm-style pass (here: part[0..G))
  GmSolve& st = S[blockIdx.x];
  double s = 0.0;
  for (int i = threadIdx.x; i < G; i += 32) s += st.part[i];
  s = warp_sum(s);
  if (threadIdx.x != 0) return;
  const double bn = sqrt(s);
  st.bnorm = bn;
  st.scale[0] = bn > 0.0 ? 1.0 / bn : 0.0;
  st.g[0] = bn;
  st.estimate = bn;
  st.target = st.target * bn;  // target holds rel_tol until here
  st.recheck_at = st.target;
  if (st.record) st.hist[0] = bn;
  if (st.max_iter == 0 && bn > 0.0) enter_finish(st, 0, st.estimate <= st.target);
}

__global__ void __launch_bounds__(256) k_bnorm_part(GmSolve* S, int G) {
  GmSolve& st = S[blockIdx.y];
  __shared__ double red[8];
  const double* b = st.V[0];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += G * blockDim.x) {
    const double v = b[vidx(i)];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += red[i];
    st.part[blockIdx.x] = t;
  }
}

// V[0] <- b in the chunk-major basis layout (b staged flat in rbuf).
__global__ void k_pack_rhs(GmSolve* S) {
  GmSolve& st = S[blockIdx.y];
  double* v0 = st.V[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += gridDim.x * blockDim.x) v0[vidx(i)] = st.rbuf[i];
}

inline unsigned cdiv(int64_t a, int64_t b) { return unsigned((a + b - 1) / b); }

// Cluster launch of the Gram-Schmidt kernels: ncl clusters of CL CTAs.
template <int CL, bool UPDATE>
cudaError_t gc_launch(cudaStream_t s, int ncl, GmSolve* S, int ns, int G, UpdSel skip) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(ncl * CL), 1u, 1u);
  cfg.blockDim = dim3(unsigned(GC_THREADS), 1u, 1u);
  cfg.dynamicSmemBytes = size_t(GC_SMEM_DOUBLES) * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(CL);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gs_clu<CL, UPDATE>, S, ns, G, skip);
}

template <int CL>
int gc_max_clusters(int sm_count) {
  const int smem = GC_SMEM_DOUBLES * int(sizeof(double));
  cudaFuncSetAttribute(k_gs_clu<CL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gs_clu<CL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(sm_count / CL * CL), 1u, 1u);
  cfg.blockDim = dim3(unsigned(GC_THREADS), 1u, 1u);
  cfg.dynamicSmemBytes = size_t(smem);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(CL);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int a = 0, b = 0;
  if (cudaOccupancyMaxActiveClusters(&a, k_gs_clu<CL, true>, &cfg) != cudaSuccess ||
      cudaOccupancyMaxActiveClusters(&b, k_gs_clu<CL, false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(std::min(a, b), sm_count / CL);
}

// Cluster size and clusters per launch of one Gram-Schmidt pass. Measured on
// C3 (k + 1 up to 335): with the plain-vector basis the projection pass was
// fastest with CTA pairs (6.3 TB/s vs 5.7), with the chunk-major basis
// unclustered (6.57 TB/s vs 6.12 for pairs); the update + probe pass is
// fastest unclustered either way (4.8 TB/s; the per-tile exchange of its row
// sums costs more than the longer tiles gain). MPG_GS_CLUSTER_DOT /
// MPG_GS_CLUSTER_UPD override (1, 2 or 4; smaller clusters are used when the
// device cannot co-schedule).
struct GcConfig {
  int cl = 1, ncl = 1;
};
GcConfig gc_config(int dev, int sm_count, bool update) {
  static std::mutex mu;
  static GcConfig cache[2][64];
  static bool have[2][64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && have[update][dev]) return cache[update][dev];
  const char* e = std::getenv(update ? "MPG_GS_CLUSTER_UPD" : "MPG_GS_CLUSTER_DOT");
  int want = e ? std::atoi(e) : 1;
  GcConfig g;
  if (want >= 4 && (g.ncl = gc_max_clusters<4>(sm_count)) > 0) g.cl = 4;
  else if (want >= 2 && (g.ncl = gc_max_clusters<2>(sm_count)) > 0) g.cl = 2;
  else {
    g.cl = 1;
    g.ncl = std::max(1, gc_max_clusters<1>(sm_count));
  }
  if (dev >= 0 && dev < 64) {
    cache[update][dev] = g;
    have[update][dev] = true;
  }
  return g;
}

cudaError_t gc_launch_any(bool update, const GcConfig& g, cudaStream_t s, GmSolve* S, int ns, int G,
                          UpdSel skip = UpdSel{0, 0, 0, 0}) {
  const UpdSel none{0, 0, 0, 0};
  (void)none;
  switch (g.cl) {
    case 4: return update ? gc_launch<4, true>(s, g.ncl, S, ns, G, skip) : gc_launch<4, false>(s, g.ncl, S, ns, G, skip);
    case 2: return update ? gc_launch<2, true>(s, g.ncl, S, ns, G, skip) : gc_launch<2, false>(s, g.ncl, S, ns, G, skip);
    default: return update ? gc_launch<1, true>(s, g.ncl, S, ns, G, skip) : gc_launch<1, false>(s, g.ncl, S, ns, G, skip);
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

// Tensor map over one basis panel, [chunks][64 vectors][16 rows] doubles, box
// of box_vecs vectors x 16 rows of one chunk, 128-byte swizzle (k_gs_tmx).
void encode_panel_map(CUtensorMap* out, double* base, int64_t chunks, int box_vecs) {
  const cuuint64_t dims[3] = {cuuint64_t(CHUNK), cuuint64_t(PANEL), cuuint64_t(chunks)};
  const cuuint64_t strides[2] = {cuuint64_t(CHUNK) * sizeof(double), cuuint64_t(PANEL * CHUNK) * sizeof(double)};
  const cuuint32_t box[3] = {cuuint32_t(CHUNK), cuuint32_t(box_vecs), 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  const CUresult r = tensor_map_encoder()(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

// Tensor map over one shadow panel, [chunks][64 vectors][32 rows] floats (k_gs_tmxf).
void encode_shadow_map(CUtensorMap* out, float* base, int64_t chunks, int box_vecs) {
  const cuuint64_t dims[3] = {cuuint64_t(FCHUNK), cuuint64_t(PANEL), cuuint64_t(chunks)};
  const cuuint64_t strides[2] = {cuuint64_t(FCHUNK) * sizeof(float), cuuint64_t(PANEL * FCHUNK) * sizeof(float)};
  const cuuint32_t box[3] = {cuuint32_t(FCHUNK), cuuint32_t(box_vecs), 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  const CUresult r = tensor_map_encoder()(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

struct SolveHost {
  std::vector<CUtensorMap> tmh;  // host mirror of the panel tensor maps (k_gs_tmx)
  DBuf<CUtensorMap> tmd;
  std::vector<CUtensorMap> tmfh;  // the same for the single-precision shadow panels (k_gs_tmxf)
  DBuf<CUtensorMap> tmfd;
  std::vector<DBuf<float>> fpanels;
  std::vector<float*> ftab;
  DBuf<float*> dF;
  std::vector<DBuf<double>> panels;
  std::vector<double*> vtab;  // host mirror of the V table
  int uploaded = 0;
  DBuf<double*> dV;
  DBuf<double> scale, h, d, H, cs, sn, g, hist, y, z0, z1, ubuf, rbuf, part, dp, hg, Hu;
  DBuf<CsrView> fac;
  int ld = 0;
};

}  // namespace

std::vector<GmresOutcome> gmres_batch(const ShiftedOp& op, std::vector<SolveSpec>& specs, const GmresOptions& opt) {
  const auto t0 = std::chrono::steady_clock::now();
  const int ns = int(specs.size());
  std::vector<GmresOutcome> out(static_cast<size_t>(ns));
  if (ns == 0) return out;
  if (opt.max_iter < 0) throw std::invalid_argument("gmres: max_iter must be nonnegative");
  const int dev = op.device;
  auto& c = ctx(dev);
  DeviceGuard guard(dev);
  cudaStream_t s = c.stream;
  const int maxit = opt.max_iter;
  const int64_t nb = op.n;

  // Per-solve dimensions and block counts.
  int64_t nmax = 0;
  for (auto& sp : specs) nmax = std::max<int64_t>(nmax, sp.sim != 0.0 ? 2 * nb : nb);
  const int ntiles = int(cdiv(nmax, DOT_TILE));
  const GcConfig gc_dot = gc_config(dev, c.sm_count, false), gc_upd = gc_config(dev, c.sm_count, true);
  // partial-sum slots per solve: the dot/update grids, and one per GS cluster
  // (>= sm_count: the persistent second pass writes one slot per SM)
  const int G = std::max(std::max(std::max(gc_dot.ncl, gc_upd.ncl), c.sm_count),
                         std::max(1, std::min(ntiles, std::max(8, (c.sm_count * 8) / ns))));

  // Update + probe kernel (MPG_GS_UPD = tmx | tma | reg): 2 = k_gs_tmx (swizzled
  // tensor copies, no per-tile barrier), 1 = k_gs_tma, 0 = register-tiled only.
  const bool fused = maxit + 1 <= UP_MAXCOLS && !std::getenv("MPG_NO_FUSE");
  // delayed second pass (DCGS2-style): a needed re-orthogonalisation of W_{k+1} is
  // applied by the next iteration's projection pass instead of its own pass over
  // the basis (MPG_DCGS2=0 restores the immediate pass)
  const bool dcgs_on = fused && !(std::getenv("MPG_DCGS2") && std::atoi(std::getenv("MPG_DCGS2")) == 0);
  // Update + probe kernels (MPG_GS_UPD = hybrid | tmx | tma | reg): k_gs_tma up
  // to k + 1 = split, k_gs_tmx above (up to GX_MAXV), the register-tiled kernel
  // beyond; measured per launch on C3.
  UpdSel usel{0, 0, 0, 0};
  if (fused && gc_upd.cl == 1) {
    const char* e = std::getenv("MPG_GS_UPD");
    usel.sel = e && !std::strcmp(e, "reg") ? 0 : e && !std::strcmp(e, "tma") ? 1 : e && !std::strcmp(e, "tmx") ? 2 : 3;
    if (!tensor_map_encoder()) usel.sel &= 1;
    const char* sp = std::getenv("MPG_GS_SPLIT");
    usel.split = sp ? std::atoi(sp) : 192;
    // the register-tiled kernel is faster for the first iterations (C3, per launch: k = 0 306 us vs 749 us for
    // k_gs_tma, k = 24 771 vs 889 us; k = 32 1 370 vs 899 us)
    const char* lo = std::getenv("MPG_GS_LOW");
    usel.low = lo ? std::atoi(lo) : 28;
  }
  UpdSel psel{0, 0, 1, 0};
  if (fused && gc_dot.cl == 1 && (usel.sel & 2)) {
    const char* e = std::getenv("MPG_GS_DOT");
    if (!(e && !std::strcmp(e, "reg"))) psel.sel = 4;
    const char* sp = std::getenv("MPG_GS_DOT_SPLIT");
    // the register-tiled projection below (C3: 192 -> 1 099 ms, 256 -> 1 074 ms, all-register 1 108 ms);
    // with the delayed second pass, which needs k_gs_tmx<true>, 128 (C3 step 3 153 -> 2 846 ms; 64: 2 864 ms)
    psel.split = sp ? std::atoi(sp) : (dcgs_on ? 128 : 256);
  }
  // single-precision shadow of the basis for the projection pass (k_gs_tmxf); needs the delayed second
  // pass, which repairs the few-digit projection coefficients (MPG_GS_F32=0: fp64 projection everywhere).
  // With it the split moves to 96 (C3 step: 128 -> 2 532 ms, 96 -> 2 497, 64 -> 2 504, 32 -> 2 526).
  const bool f32_on = dcgs_on && (psel.sel & 4) && !(std::getenv("MPG_GS_F32") && std::atoi(std::getenv("MPG_GS_F32")) == 0);
  // re-swept after the k_gs_tmxf rework: 96 -> 2 220, 64 / 48 -> 2 195, 32 -> 2 202 ms per C3 step. 96 stays: the
  // 1 % is not worth re-deciding the rounding-determined trajectory of the C2 BASELINE-seed IRKA (
  // with 64 the unmirrored reference loop meets an unstable pole in sweep 3 and raises the reference's SolverError)
  if (f32_on && !std::getenv("MPG_GS_DOT_SPLIT")) psel.split = 96;
  // k_gs_tmxf: from this many 8-vector boxes on, the last shadow panel is fetched whole (gf_split; 9: never)
  psel.low = std::getenv("MPG_GF_MBFULL") ? std::atoi(std::getenv("MPG_GF_MBFULL")) : 5;
  // ... and (bits 8 up) the most vectors for which a consumer step covers two chunks (MPG_GF_CF2MAX <= 256)
  psel.low = (psel.low & 0xff) |
             (std::min(256, std::getenv("MPG_GF_CF2MAX") ? std::atoi(std::getenv("MPG_GF_CF2MAX")) : 224) << 8);  // 192 / 224 / 256: gs_dot 716 / 694 / 700 ms per C3 step
  const int upd_kind = usel.sel;
  const bool want_maps = ((usel.sel | psel.sel) & 6) != 0;  // panel tensor maps for k_gs_tmx
  std::vector<SolveHost> sh(static_cast<size_t>(ns));
  std::vector<GmSolve> hs(static_cast<size_t>(ns));
  int max_stages = 0;
  double max_fac_mean = 0.0;
  int64_t max_fac_rows = 0;
  int max_fac_bblk = 0;  // row-binned factors (irregular rows): the largest binned grid
  bool any_fac_plain = false;
  for (int i = 0; i < ns; ++i) {
    SolveSpec& sp = specs[size_t(i)];
    SolveHost& H = sh[size_t(i)];
    GmSolve& g = hs[size_t(i)];
    std::memset(&g, 0, sizeof g);
    const bool pair = sp.sim != 0.0;
    const int64_t n = pair ? 2 * nb : nb;
    if (sp.chain) {
      const int64_t fdim = sp.chain->factors[0]->nrows;
      if (!(fdim == n || (pair && fdim == nb)))
        throw std::invalid_argument("gmres: preconditioner dimension does not match the system");
      sp.pair_blockdiag = pair && fdim == nb;
      for (auto& f : sp.chain->factors)
        if (f->device != dev) throw std::invalid_argument("gmres: preconditioner on a different device");
    }
    g.n = int(n);
    g.nbase = int(nb);
    g.pair = pair;
    g.transpose = sp.transpose;
    g.sre = sp.sre;
    g.sim = sp.sim;
    g.ca = sp.ca;
    g.stages = sp.chain ? int(sp.chain->factors.size()) : 0;
    g.pair_bd = sp.pair_blockdiag;
    g.max_iter = maxit;
    g.record = opt.record_history;
    g.target = opt.rel_tol;  // scaled by bnorm in k_init
    g.phase = PH_RUN;
    H.ld = int((n + 31) / 32 * 32);  // rows per panel (multiple of the 16-row chunk)
    H.dV = DBuf<double*>(dev, size_t(maxit) + 2);
    H.vtab.assign(size_t(maxit) + 2, nullptr);
    const size_t m1 = size_t(maxit) + 2;
    H.scale = DBuf<double>(dev, m1);
    H.h = DBuf<double>(dev, m1);
    H.d = DBuf<double>(dev, m1);
    H.H = DBuf<double>(dev, std::max<size_t>(1, size_t(maxit) * size_t(maxit + 1) / 2));
    H.cs = DBuf<double>(dev, m1);
    H.sn = DBuf<double>(dev, m1);
    H.g = DBuf<double>(dev, m1);
    H.hist = DBuf<double>(dev, m1);
    H.y = DBuf<double>(dev, m1);
    H.z0 = DBuf<double>(dev, size_t(H.ld));
    H.z1 = DBuf<double>(dev, size_t(H.ld));
    H.ubuf = DBuf<double>(dev, size_t(H.ld));
    H.rbuf = DBuf<double>(dev, size_t(H.ld));
    H.part = DBuf<double>(dev, m1 * size_t(G));
    H.dp = DBuf<double>(dev, m1);
    H.hg = DBuf<double>(dev, m1);
    H.Hu = DBuf<double>(dev, std::max<size_t>(1, hoff2(maxit)));
    MPG_CUDA(cudaMemsetAsync(H.g.get(), 0, m1 * sizeof(double), s));
    if (g.stages) {
      std::vector<CsrView> fv;
      for (auto& f : sp.chain->factors) {
        fv.push_back(f->view());
        if (f->brow.get()) {
          max_fac_bblk = std::max(max_fac_bblk, f->bblk[NBIN]);
          continue;
        }
        any_fac_plain = true;
        max_fac_mean = std::max(max_fac_mean, f->mean_row);
        max_fac_rows = std::max<int64_t>(max_fac_rows, f->nrows * (g.pair_bd ? 2 : 1));
      }
      H.fac = DBuf<CsrView>(dev, fv.size());
      MPG_CUDA(cudaMemcpyAsync(H.fac.get(), fv.data(), fv.size() * sizeof(CsrView), cudaMemcpyHostToDevice, s));
      max_stages = std::max(max_stages, g.stages);
    }
    g.V = H.dV.get();
    g.scale = H.scale.get();
    g.h = H.h.get();
    g.d = H.d.get();
    g.H = H.H.get();
    g.cs = H.cs.get();
    g.sn = H.sn.get();
    g.g = H.g.get();
    g.hist = H.hist.get();
    g.y = H.y.get();
    g.z0 = H.z0.get();
    g.z1 = H.z1.get();
    g.ubuf = H.ubuf.get();
    g.rbuf = H.rbuf.get();
    g.part = H.part.get();
    g.fac = H.fac.get();
    g.dp = H.dp.get();
    g.hg = H.hg.get();
    g.Hu = H.Hu.get();
    g.dcgs = dcgs_on ? 1 : 0;
    g.pend = 0;
    if (want_maps) {
      const size_t np = size_t(maxit + 2 + PANEL - 1) / PANEL;
      H.tmh.resize(2 * np);
      H.tmd = DBuf<CUtensorMap>(dev, 2 * np);
      g.tm = H.tmd.get();
      if (f32_on) {
        H.tmfh.resize(2 * np);
        H.tmfd = DBuf<CUtensorMap>(dev, 2 * np);
        g.tmf = H.tmfd.get();
        H.dF = DBuf<float*>(dev, size_t(maxit) + 2);
        H.ftab.assign(size_t(maxit) + 2, nullptr);
        g.F = H.dF.get();
      }
    }
  }

  // Basis panels: make vectors [0, upto) available for solve i.
  auto ensure = [&](int i, int upto) {
    SolveHost& H = sh[size_t(i)];
    upto = std::min(upto, maxit + 2);
    while (int(H.panels.size()) * PANEL < upto) {
      H.panels.emplace_back(dev, size_t(PANEL) * size_t(H.ld));
      double* base = H.panels.back().get();
      // padding rows are read (as zeros) by the Gram-Schmidt tiles
      MPG_CUDA(cudaMemsetAsync(base, 0, size_t(PANEL) * size_t(H.ld) * sizeof(double), s));
      const int p0 = int(H.panels.size() - 1) * PANEL;
      for (int j = 0; j < PANEL && p0 + j < maxit + 2; ++j) H.vtab[size_t(p0 + j)] = base + size_t(j) * CHUNK;
      if (want_maps) {
        const size_t p = H.panels.size() - 1;
        encode_panel_map(&H.tmh[2 * p], base, H.ld / CHUNK, PANEL);
        encode_panel_map(&H.tmh[2 * p + 1], base, H.ld / CHUNK, 8);
        MPG_CUDA(cudaMemcpyAsync(H.tmd.get() + 2 * p, &H.tmh[2 * p], 2 * sizeof(CUtensorMap), cudaMemcpyHostToDevice, s));
      }
      if (hs[size_t(i)].F) {
        H.fpanels.emplace_back(dev, size_t(PANEL) * size_t(H.ld));
        float* fb = H.fpanels.back().get();
        MPG_CUDA(cudaMemsetAsync(fb, 0, size_t(PANEL) * size_t(H.ld) * sizeof(float), s));
        for (int j = 0; j < PANEL && p0 + j < maxit + 2; ++j) H.ftab[size_t(p0 + j)] = fb + size_t(j) * FCHUNK;
        const size_t p = H.fpanels.size() - 1;
        encode_shadow_map(&H.tmfh[2 * p], fb, H.ld / FCHUNK, PANEL);
        encode_shadow_map(&H.tmfh[2 * p + 1], fb, H.ld / FCHUNK, 8);
        MPG_CUDA(cudaMemcpyAsync(H.tmfd.get() + 2 * p, &H.tmfh[2 * p], 2 * sizeof(CUtensorMap), cudaMemcpyHostToDevice, s));
      }
    }
    if (upto > H.uploaded) {
      if (hs[size_t(i)].F)
        MPG_CUDA(cudaMemcpyAsync(H.dF.get() + H.uploaded, H.ftab.data() + H.uploaded,
                                 size_t(upto - H.uploaded) * sizeof(float*), cudaMemcpyHostToDevice, s));
      MPG_CUDA(cudaMemcpyAsync(H.dV.get() + H.uploaded, H.vtab.data() + H.uploaded,
                               size_t(upto - H.uploaded) * sizeof(double*), cudaMemcpyHostToDevice, s));
      H.uploaded = upto;
    }
  };

  for (int i = 0; i < ns; ++i) {
    ensure(i, std::min(maxit + 2, 2));
    copy_in(sh[size_t(i)].rbuf.get(), specs[size_t(i)].b, size_t(hs[size_t(i)].n), s);
  }
  DBuf<GmSolve> dS(dev, size_t(ns));
  MPG_CUDA(cudaMemcpyAsync(dS.get(), hs.data(), sizeof(GmSolve) * size_t(ns), cudaMemcpyHostToDevice, s));
  k_pack_rhs<<<dim3(unsigned(std::min<int64_t>(cdiv(nmax, 256), 4096)), unsigned(ns)), 256, 0, s>>>(dS.get());
  MPG_CHECK_LAUNCH();
  count_launch();
  k_bnorm_part<<<dim3(unsigned(G), unsigned(ns)), 256, 0, s>>>(dS.get(), G);
  MPG_CHECK_LAUNCH();
  k_init<<<unsigned(ns), 32, 0, s>>>(dS.get(), G);
  MPG_CHECK_LAUNCH();
  count_launch(2);
  MPG_CUDA(cudaMemcpyAsync(hs.data(), dS.get(), sizeof(GmSolve) * size_t(ns), cudaMemcpyDeviceToHost, s));
  MPG_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < ns; ++i)
    if (hs[size_t(i)].bnorm == 0.0) throw std::invalid_argument("gmres: zero right-hand side");

  // ---- capture one iteration (plus the conditional assembly) as a graph ----
  const OpView opn = op.view(false), opt_ = op.view(true);
  const int Vop = op.vec_width;
  const int Vfac = choose_vec_width(max_fac_mean);
  const size_t smem_dot = size_t(DOT_TILE + maxit + 2) * sizeof(double);
  const size_t smem_upd = size_t(2 * (maxit + 2)) * sizeof(double);
  // Dynamic shared-memory opt-ins are per device context: set them once per
  // device (the library keeps one context per device, ctx(dev)).
  {
    static std::mutex attr_mu;
    static std::set<int> attr_done;
    std::lock_guard<std::mutex> lk(attr_mu);
    if (attr_done.insert(op.device).second) {
      cudaFuncSetAttribute(k_dot, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_backsub, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_reorth_p, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      // TMA-staged update + probe kernels: slots = the update clusters, one CTA each.
      cudaFuncSetAttribute(k_gs_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, GT_SMEM);
      cudaFuncSetAttribute(k_gs_tmx<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GX_SMEM);
      cudaFuncSetAttribute(k_gs_tmx<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GX_SMEM);
      cudaFuncSetAttribute(k_gs_tmxf, cudaFuncAttributeMaxDynamicSharedMemorySize, GF_SMEM);
      cudaFuncSetAttribute(k_spmv_sell8t<E_IDENT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(k_spmv_sell8t<E_IDENT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(k_spmv_sell8t<E_DIAG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(k_spmv_sell8t<E_SAMEPAT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);

      if (const char* co = std::getenv("MPG_SELL_CARVEOUT")) {  // shared-memory share of the unified L1 (percent)
        const int pc = std::atoi(co);
        cudaFuncSetAttribute(k_spmv_sell8t<E_IDENT, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
        cudaFuncSetAttribute(k_spmv_sell8t<E_IDENT, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
        cudaFuncSetAttribute(k_spmv_sell8t<E_DIAG, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
        cudaFuncSetAttribute(k_spmv_sell8t<E_SAMEPAT, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
      }
      const int hsm = HALO_MAX * HALO_XSTRIDE * int(sizeof(double2));
      cudaFuncSetAttribute(k_spmv_halo<E_IDENT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
      cudaFuncSetAttribute(k_spmv_halo<E_IDENT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
      cudaFuncSetAttribute(k_spmv_halo<E_DIAG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
      cudaFuncSetAttribute(k_spmv_halo<E_SAMEPAT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
    }
  }
  const bool need_reg_upd = upd_kind == 0 || usel.low > 0 || (upd_kind == 1 && maxit + 1 > GT_MAXCOLS) ||
                            ((upd_kind & 2) && maxit + 2 > GX_MAXV);
  const bool need_tma = (upd_kind & 1) && (upd_kind == 1 || usel.split > 0);
  const bool need_tmx = (upd_kind & 2) && (upd_kind == 2 || maxit + 1 > usel.split);
  const size_t smem_ro = size_t(2 * UP_MAXCOLS + 32) * sizeof(double) + size_t(ns) * sizeof(int);
  int launches_per_iter = 0;
  // Profiling hook: called after every launch with a kernel-class id.
  std::function<void(int)> mark = [](int) {};
  // Shared-matrix groups (MPG_NO_MULTI disables): solves with the same chain
  // (non-pair) and real shifts on the same operator side.
  std::vector<Group> chain_groups, op_groups_run, op_groups_asm;
  std::vector<const Chain*> chain_of_group;
  std::vector<char> chain_il;          // chain group runs the interleaved path in run mode
  std::vector<Group> il_groups;        // per chain group: its columns on that path (the group + complex pairs riding along)
  std::vector<DBuf<double>> il_bufs;   // two [n][MB] buffers per chain group (empty if not il)
  bool any_plain_chain = true, any_plain_op_run = true, any_plain_op_asm = true;
  // The solves the plain (per-solve) chain / operator launches serve, per mode: blockIdx.y walks these lists,
  // so a batch whose solves are all advanced by group kernels launches nothing, and a few ungrouped solves
  // (complex pairs in assembly mode) do not cost a grid over the whole batch.
  std::vector<int> pl_chain[2], pl_op[2];
  DBuf<int> pl_buf(dev, size_t(4 * ns));
  auto build_plain_lists = [&]() {
    for (int m = 0; m < 2; ++m) { pl_chain[m].clear(); pl_op[m].clear(); }
    for (int i = 0; i < ns; ++i) {
      const GmSolve& m = hs[size_t(i)];
      if (m.stages > 0 && !m.grouped_chain) {
        if (!m.il_run) pl_chain[0].push_back(i);
        pl_chain[1].push_back(i);
      }
      if (!(m.grouped_op & 1)) pl_op[0].push_back(i);
      if (!(m.grouped_op & 2)) pl_op[1].push_back(i);
    }
    std::vector<int> flat(size_t(4 * ns), 0);
    for (int m = 0; m < 2; ++m) {
      std::copy(pl_chain[m].begin(), pl_chain[m].end(), flat.begin() + size_t(m) * ns);
      std::copy(pl_op[m].begin(), pl_op[m].end(), flat.begin() + size_t(2 + m) * ns);
    }
    MPG_CUDA(cudaMemcpyAsync(pl_buf.get(), flat.data(), flat.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    MPG_CUDA(cudaStreamSynchronize(s));  // flat is a local
  };
  bool il2 = false;  // RHS-split interleaved SpMVs
  bool use_halo = false;
  bool use_sell = false;
  // SELL-8 kernels with the matrix stream staged by TMA bulk copies (MPG_SELL_TMA=0: plain loads)
  const bool sell_tma = !(std::getenv("MPG_SELL_TMA") && std::atoi(std::getenv("MPG_SELL_TMA")) == 0);
  // row-binned interleaved SpMV for irregular matrices (MPG_IL_BINS=0: the fixed four lanes per row)
  const bool il_bins = !(std::getenv("MPG_IL_BINS") && std::atoi(std::getenv("MPG_IL_BINS")) == 0);
  // SM-affine persistent SELL-8 kernels (MPG_SELL_PERSIST=1; CTAs per SM: MPG_SELL_OCC)
  DBuf<int> sell_ctr_buf;
  int* sell_ctr = nullptr;
  const int sell_occ = std::getenv("MPG_SELL_OCC") ? std::max(1, std::atoi(std::getenv("MPG_SELL_OCC"))) : 8;
  // measured slower on C3 (step 2 519 -> 2 793 / 2 750 / 2 947 ms with 8 / 6 / 4 CTAs per SM): opt-in
  if (std::getenv("MPG_SELL_PERSIST") && std::atoi(std::getenv("MPG_SELL_PERSIST")) != 0) {
    sell_ctr_buf = DBuf<int>(dev, size_t(c.sm_count) + 1);
    MPG_CUDA(cudaMemsetAsync(sell_ctr_buf.get(), 0, (size_t(c.sm_count) + 1) * sizeof(int), s));
    sell_ctr = sell_ctr_buf.get();
  }
  if (!std::getenv("MPG_NO_MULTI")) {
    std::vector<int> used(size_t(ns), 0);
    for (int i = 0; i < ns; ++i) {
      if (used[size_t(i)] || !specs[size_t(i)].chain || hs[size_t(i)].pair_bd) continue;
      std::vector<int> mem{i};
      for (int j = i + 1; j < ns; ++j)
        if (!used[size_t(j)] && specs[size_t(j)].chain && !hs[size_t(j)].pair_bd &&
            specs[size_t(j)].chain->factors == specs[size_t(i)].chain->factors)
          mem.push_back(j);
      if (mem.size() < 2) continue;
      for (size_t b = 0; b < mem.size(); b += MB) {
        Group g{};
        g.cnt = int(std::min<size_t>(MB, mem.size() - b));
        for (int q = 0; q < g.cnt; ++q) g.idx[q] = mem[b + size_t(q)];
        chain_groups.push_back(g);
        chain_of_group.push_back(specs[size_t(i)].chain.get());
      }
      for (int m : mem) { used[size_t(m)] = 1; hs[size_t(m)].grouped_chain = 1; }
    }
    // interleaved path: chain groups of real shifts on one operator side
    const bool il_on = !std::getenv("MPG_NO_IL");
    il2 = std::getenv("MPG_IL_NNZSPLIT") == nullptr;  // RHS split measured faster (C3: 256 -> 221 ms / 348 its)
    // halo-staged sliced ELL: opt-in (MPG_SPMV_HALO=1); measured slower than the
    // CSR kernels on C3 (operator 309 -> 398-463 us, chain 168 -> 288 us per launch)
    use_halo = std::getenv("MPG_SPMV_HALO") != nullptr && std::getenv("MPG_SPMV_CSR") == nullptr;
    use_sell = !use_halo && std::getenv("MPG_SPMV_CSR") == nullptr;  // SELL-8 where the padding stays small
    std::vector<int> in_il(size_t(ns), 0);
    for (size_t gi = 0; gi < chain_groups.size(); ++gi) {
      const Group& g = chain_groups[gi];
      bool ok = il_on && g.cnt >= 2;
      for (int q = 0; q < g.cnt && ok; ++q) {
        const GmSolve& m = hs[size_t(g.idx[q])];
        ok = !m.pair && m.transpose == hs[size_t(g.idx[0])].transpose && m.n == int(nb);
      }
      chain_il.push_back(ok ? 1 : 0);
      if (ok && use_halo) {  // build the halo layouts now: the iteration is captured into a graph
        for (const CsrPtr& f : chain_of_group[gi]->factors) halo_of(*f, nullptr);
        halo_of_op(op, hs[size_t(g.idx[0])].transpose != 0, nullptr);
      }
      if (ok && use_sell) {
        for (const CsrPtr& f : chain_of_group[gi]->factors) sell_of(*f, nullptr);
        sell_of_op(op, hs[size_t(g.idx[0])].transpose != 0, nullptr);
      }
      Group ig = g;  // the group as the interleaved launches see it
      ig.hm = 0;
      if (ok) {
        il_bufs.emplace_back(dev, size_t(nb) * MB);
        il_bufs.emplace_back(dev, size_t(nb) * MB);
        for (int q = 0; q < g.cnt; ++q) in_il[size_t(g.idx[q])] = 1;
        // Complex pairs of the same side and chain ride along as two columns each (placed first, so they
        // start at even columns): their chain and operator SpMVs then cost nothing beyond the group's own
        // launches (C3 IRKA: 4 real + 2 pair units per side from sweep 3 on fill the 8 columns). Only on
        // the TMA-staged SELL-8 path, whose epilogue knows the pair coupling.
        const bool tr = hs[size_t(g.idx[0])].transpose != 0;
        bool pairs_ok = use_sell && sell_tma && !std::getenv("MPG_NO_IL_PAIRS");
        if (pairs_ok) {
          for (const CsrPtr& f : chain_of_group[gi]->factors) {
            const Sell8* p8 = sell_of(*f, nullptr);
            pairs_ok = pairs_ok && p8 && size_t(p8->max_tile) * 12 <= 64 * 1024;
          }
          const Sell8* o8 = sell_of_op(op, tr, nullptr);
          pairs_ok = pairs_ok && o8 && size_t(o8->max_tile) * (op.emode == E_SAMEPAT ? 20 : 12) <= 64 * 1024;
        }
        std::vector<int> prs;
        if (pairs_ok)
          for (int j = 0; j < ns && int(prs.size()) < (MB - g.cnt) / 2; ++j) {
            const GmSolve& m = hs[size_t(j)];
            if (m.pair && m.pair_bd && !in_il[size_t(j)] && specs[size_t(j)].chain && (m.transpose != 0) == tr &&
                m.n == 2 * int(nb) && specs[size_t(j)].chain->factors == chain_of_group[gi]->factors)
              prs.push_back(j);
          }
        if (!prs.empty()) {
          Group ng{};
          int c = 0;
          for (int j : prs) {
            ng.idx[c] = j; ng.set_half(c++, 1);
            ng.idx[c] = j; ng.set_half(c++, 2);
            in_il[size_t(j)] = 1;
            hs[size_t(j)].il_run = 1;
          }
          for (int q = 0; q < g.cnt; ++q) ng.idx[c++] = g.idx[q];
          ng.cnt = c;
          ig = ng;
        }
        // the same condition (every launch of the group on the TMA-staged SELL-8 path) allows the narrow mode
        bool t8 = use_sell && sell_tma && !std::getenv("MPG_NO_IL_NARROW");
        if (t8) {
          for (const CsrPtr& f : chain_of_group[gi]->factors) {
            const Sell8* p8 = sell_of(*f, nullptr);
            t8 = t8 && p8 && size_t(p8->max_tile) * 12 <= 64 * 1024;
          }
          const Sell8* o8 = sell_of_op(op, tr, nullptr);
          t8 = t8 && o8 && size_t(o8->max_tile) * (op.emode == E_SAMEPAT ? 20 : 12) <= 64 * 1024;
        }
        if (t8) ig.hm |= 1u << 31;
      } else {
        il_bufs.emplace_back();
        il_bufs.emplace_back();
      }
      il_groups.push_back(ig);
    }
    for (int mode = 0; mode < 2; ++mode)
      for (int side = 0; side < 2; ++side) {
        std::vector<int> mem;
        for (int i = 0; i < ns; ++i)
          if (!hs[size_t(i)].pair && hs[size_t(i)].transpose == side && !(mode == 0 && in_il[size_t(i)]))
            mem.push_back(i);
        if (mem.size() < 2) continue;
        for (size_t b = 0; b < mem.size(); b += MB) {
          Group g{};
          g.cnt = int(std::min<size_t>(MB, mem.size() - b));
          for (int q = 0; q < g.cnt; ++q) g.idx[q] = mem[b + size_t(q)];
          (mode == 0 ? op_groups_run : op_groups_asm).push_back(g);
        }
        for (int m : mem) hs[size_t(m)].grouped_op |= mode == 0 ? 1 : 2;
      }
    for (int i = 0; i < ns; ++i)
      if (in_il[size_t(i)]) hs[size_t(i)].grouped_op |= 1;
    any_plain_chain = any_plain_op_run = any_plain_op_asm = false;
    for (int i = 0; i < ns; ++i) {
      const GmSolve& m = hs[size_t(i)];
      if (m.stages > 0 && !m.grouped_chain) any_plain_chain = true;
      if (!(m.grouped_op & 1)) any_plain_op_run = true;
      if (!(m.grouped_op & 2)) any_plain_op_asm = true;
    }
    MPG_CUDA(cudaMemcpyAsync(dS.get(), hs.data(), sizeof(GmSolve) * size_t(ns), cudaMemcpyHostToDevice, s));
  }
  build_plain_lists();
  auto chain_stage = [&](int stage, int mode) {
    for (size_t gi = 0; gi < chain_groups.size(); ++gi) {
      const Chain& ch = *chain_of_group[gi];
      if (stage >= int(ch.factors.size())) continue;
      const DevCsr& f = *ch.factors[size_t(stage)];
      const int Vf = choose_vec_width(f.mean_row);
      const unsigned grid = cdiv(f.nrows * int64_t(Vf), 256);
      if (mode == 0 && chain_il[gi]) {
        double* xa = il_bufs[2 * gi].get();
        double* xb = il_bufs[2 * gi + 1].get();
        if (stage == 0) {
          k_pack_il<<<cdiv(nb * MB, 256), 256, 0, s>>>(dS.get(), il_groups[gi], xa, int(nb));
          ++launches_per_iter;
          mark(PK_CHAIN);
        }
        const double* xin = (stage & 1) ? xb : xa;
        double* xout = (stage & 1) ? xa : xb;
        Sell8View sv{};
        const Sell8* sp8 = use_sell ? sell_of(f, &sv) : nullptr;
        if (sp8) {
          if (sell_tma && size_t(sp8->max_tile) * 12 <= 64 * 1024)
            k_spmv_sell8t<E_IDENT, true><<<cdiv(cdiv(f.nrows, 8), 8), 256, size_t(sp8->max_tile) * 12, s>>>(
                dS.get(), il_groups[gi], sv, opn, xin, xout);
          else if (sell_ctr)
            k_spmv_sell8p<E_IDENT, true><<<unsigned(c.sm_count * sell_occ), 256, 0, s>>>(dS.get(), il_groups[gi], sv, opn,
                                                                                     xin, xout, sell_ctr, c.sm_count);
          else
          k_spmv_sell8<E_IDENT, true><<<cdiv(f.nrows * 4, 256), 256, 0, s>>>(dS.get(), il_groups[gi], sv, opn, xin,
                                                                          xout);
          ++launches_per_iter;
          mark(PK_CHAIN);
          continue;
        }
        HaloView hv{};
        const HaloPattern* hp = use_halo ? halo_of(f, &hv) : nullptr;
        if (hp) {
          k_spmv_halo<E_IDENT, true><<<hp->nblocks, 4 * HALO_R, size_t(hp->max_halo) * HALO_XSTRIDE * sizeof(double2), s>>>(
              dS.get(), il_groups[gi], hv, opn, xin, xout);
          ++launches_per_iter;
          mark(PK_CHAIN);
          continue;
        }
        if (il2 && f.brow.get() && il_bins) {
          unsigned gb = 0;
          for (int b = 0; b < NBIN; ++b) gb += unsigned(il2b_blocks(f.boff, b));
          k_spmv_il2b<E_IDENT, true><<<gb, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), opn, xin, xout);
          ++launches_per_iter;
          mark(PK_CHAIN);
          continue;
        }
        if (il2) {
          k_spmv_il2<E_IDENT, true><<<cdiv(f.nrows * 4, 256), 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), opn,
                                                                         xin, xout);
          ++launches_per_iter;
          mark(PK_CHAIN);
          continue;
        }
        switch (Vf) {
          case 2: k_chain_il<2><<<grid, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), xin, xout); break;
          case 4: k_chain_il<4><<<grid, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), xin, xout); break;
          case 8: k_chain_il<8><<<grid, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), xin, xout); break;
          case 16: k_chain_il<16><<<grid, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), xin, xout); break;
          default: k_chain_il<32><<<grid, 256, 0, s>>>(dS.get(), il_groups[gi], f.view(), xin, xout); break;
        }
        ++launches_per_iter;
        mark(PK_CHAIN);
        continue;
      }
      const unsigned gridm = mode == 0 ? grid : std::min<unsigned>(grid, unsigned(c.sm_count) * 8u);
      switch (Vf) {
        case 2: k_chain_multi<2><<<gridm, 256, 0, s>>>(dS.get(), chain_groups[gi], f.view(), stage, mode); break;
        case 4: k_chain_multi<4><<<gridm, 256, 0, s>>>(dS.get(), chain_groups[gi], f.view(), stage, mode); break;
        case 8: k_chain_multi<8><<<gridm, 256, 0, s>>>(dS.get(), chain_groups[gi], f.view(), stage, mode); break;
        case 16: k_chain_multi<16><<<gridm, 256, 0, s>>>(dS.get(), chain_groups[gi], f.view(), stage, mode); break;
        default: k_chain_multi<32><<<gridm, 256, 0, s>>>(dS.get(), chain_groups[gi], f.view(), stage, mode); break;
      }
      ++launches_per_iter;
      mark(mode == 0 ? PK_CHAIN : PK_ASM);
    }
    if (!any_plain_chain || pl_chain[mode].empty()) return;
    const int* lp = pl_buf.get() + size_t(mode) * ns;
    const unsigned ny = unsigned(pl_chain[mode].size());
    if (max_fac_bblk) {
      if (stage == 0 && mode == 0) {
        k_unchunk<<<dim3(unsigned(std::min<int64_t>(cdiv(nmax, 256), 2368)), ny), 256, 0, s>>>(dS.get(), lp);
        ++launches_per_iter;
        mark(PK_CHAIN);
      }
      k_chain_stage<0><<<dim3(unsigned(max_fac_bblk), ny), 256, 0, s>>>(dS.get(), stage, mode, lp);
      ++launches_per_iter;
      mark(mode == 0 ? PK_CHAIN : PK_ASM);
    }
    if (!any_fac_plain) return;
    const unsigned gfull = cdiv(max_fac_rows * int64_t(Vfac), 256);
    const dim3 grid(mode == 0 ? gfull : std::min<unsigned>(gfull, unsigned(c.sm_count) * 8u), ny);
    switch (Vfac) {
      case 2: k_chain_stage<2><<<grid, 256, 0, s>>>(dS.get(), stage, mode, lp); break;
      case 4: k_chain_stage<4><<<grid, 256, 0, s>>>(dS.get(), stage, mode, lp); break;
      case 8: k_chain_stage<8><<<grid, 256, 0, s>>>(dS.get(), stage, mode, lp); break;
      case 16: k_chain_stage<16><<<grid, 256, 0, s>>>(dS.get(), stage, mode, lp); break;
      default: k_chain_stage<32><<<grid, 256, 0, s>>>(dS.get(), stage, mode, lp); break;
    }
    ++launches_per_iter;
    mark(mode == 0 ? PK_CHAIN : PK_ASM);
  };
  auto iter_op = [&](int mode) {
    if (mode == 0)
      for (size_t gi = 0; gi < chain_groups.size(); ++gi) {
        if (!chain_il[gi]) continue;
        const Group& g = il_groups[gi];
        const OpView& ov = hs[size_t(g.idx[0])].transpose ? opt_ : opn;
        const int nst = int(chain_of_group[gi]->factors.size());
        const double* xin = ((nst - 1) & 1) ? il_bufs[2 * gi].get() : il_bufs[2 * gi + 1].get();
        const unsigned grid1 = cdiv(nb * int64_t(Vop), 256);
        Sell8View sv{};
        const Sell8* sp8 = use_sell ? sell_of_op(op, hs[size_t(g.idx[0])].transpose != 0, &sv) : nullptr;
        if (sp8) {
          const unsigned g2 = cdiv(nb * 4, 256);
          switch (op.emode) {
#define MPG_S8(EMV)                                                                                                  \
  if (sell_tma && size_t(sp8->max_tile) * (EMV == E_SAMEPAT ? 20 : 12) <= 64 * 1024)                                 \
    k_spmv_sell8t<EMV, false><<<cdiv(cdiv(nb, 8), 8), 256, size_t(sp8->max_tile) * (EMV == E_SAMEPAT ? 20 : 12), s>>>( \
        dS.get(), g, sv, ov, xin, nullptr);                                                                          \
  else if (sell_ctr)                                                                                                 \
    k_spmv_sell8p<EMV, false><<<unsigned(c.sm_count * sell_occ), 256, 0, s>>>(dS.get(), g, sv, ov, xin, nullptr, sell_ctr, \
                                                                            c.sm_count);                           \
  else                                                                                                               \
    k_spmv_sell8<EMV, false><<<g2, 256, 0, s>>>(dS.get(), g, sv, ov, xin, nullptr);
            case E_IDENT: MPG_S8(E_IDENT) break;
            case E_DIAG: MPG_S8(E_DIAG) break;
            default: MPG_S8(E_SAMEPAT) break;
#undef MPG_S8
          }
          ++launches_per_iter;
          mark(PK_OP);
          continue;
        }
        HaloView hv{};
        const HaloPattern* hp = use_halo ? halo_of_op(op, hs[size_t(g.idx[0])].transpose != 0, &hv) : nullptr;
        if (hp) {
          const size_t sm = size_t(hp->max_halo) * HALO_XSTRIDE * sizeof(double2);
          switch (op.emode) {
            case E_IDENT: k_spmv_halo<E_IDENT, false><<<hp->nblocks, 4 * HALO_R, sm, s>>>(dS.get(), g, hv, ov, xin, nullptr); break;
            case E_DIAG: k_spmv_halo<E_DIAG, false><<<hp->nblocks, 4 * HALO_R, sm, s>>>(dS.get(), g, hv, ov, xin, nullptr); break;
            default: k_spmv_halo<E_SAMEPAT, false><<<hp->nblocks, 4 * HALO_R, sm, s>>>(dS.get(), g, hv, ov, xin, nullptr); break;
          }
          ++launches_per_iter;
          mark(PK_OP);
          continue;
        }
        if (il2 && ov.a.brow && il_bins) {
          const CsrView none{};
          unsigned gb = 0;
          for (int b = 0; b < NBIN; ++b) gb += unsigned(il2b_blocks(ov.a.boff, b));
          switch (op.emode) {
            case E_IDENT: k_spmv_il2b<E_IDENT, false><<<gb, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
            case E_DIAG: k_spmv_il2b<E_DIAG, false><<<gb, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
            default: k_spmv_il2b<E_SAMEPAT, false><<<gb, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
          }
          ++launches_per_iter;
          mark(PK_OP);
          continue;
        }
        if (il2) {
          const CsrView none{};
          const unsigned g2 = cdiv(nb * 4, 256);
          switch (op.emode) {
            case E_IDENT: k_spmv_il2<E_IDENT, false><<<g2, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
            case E_DIAG: k_spmv_il2<E_DIAG, false><<<g2, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
            default: k_spmv_il2<E_SAMEPAT, false><<<g2, 256, 0, s>>>(dS.get(), g, none, ov, xin, nullptr); break;
          }
          ++launches_per_iter;
          mark(PK_OP);
          continue;
        }
#define MPG_OPI(VV)                                                                                            \
  switch (op.emode) {                                                                                          \
    case E_IDENT: k_op_il<VV, E_IDENT><<<grid1, 256, 0, s>>>(dS.get(), g, ov, xin); break;                    \
    case E_DIAG: k_op_il<VV, E_DIAG><<<grid1, 256, 0, s>>>(dS.get(), g, ov, xin); break;                      \
    default: k_op_il<VV, E_SAMEPAT><<<grid1, 256, 0, s>>>(dS.get(), g, ov, xin); break;                       \
  }
        switch (Vop) {
          case 2: MPG_OPI(2); break;
          case 4: MPG_OPI(4); break;
          case 8: MPG_OPI(8); break;
          case 16: MPG_OPI(16); break;
          default: MPG_OPI(32); break;
        }
#undef MPG_OPI
        ++launches_per_iter;
        mark(PK_OP);
      }
    const int* olp = pl_buf.get() + size_t(2 + mode) * ns;
    const unsigned ony = unsigned(std::max<size_t>(1, pl_op[mode].size()));
    const unsigned ogfull = cdiv(nb * int64_t(Vop), 256);
    const dim3 grid(mode == 0 ? ogfull : std::min<unsigned>(ogfull, unsigned(c.sm_count) * 8u), ony);
#define MPG_OPL(VV)                                                                                            \
  switch (op.emode) {                                                                                          \
    case E_IDENT: k_iter_op<VV, E_IDENT><<<grid, 256, 0, s>>>(dS.get(), opn, opt_, mode, olp); break;         \
    case E_DIAG: k_iter_op<VV, E_DIAG><<<grid, 256, 0, s>>>(dS.get(), opn, opt_, mode, olp); break;           \
    default: k_iter_op<VV, E_SAMEPAT><<<grid, 256, 0, s>>>(dS.get(), opn, opt_, mode, olp); break;            \
  }
    if ((mode == 0 ? any_plain_op_run : any_plain_op_asm) && !pl_op[mode].empty()) {
      // the sides present among the solves, split by row-binned / plain operator rows
      bool need_b = false, need_p = false;
      for (int i : pl_op[mode]) ((hs[size_t(i)].transpose ? opt_ : opn).a.brow ? need_b : need_p) = true;
      if (need_b) {
        const dim3 grid(unsigned(std::max(opn.a.brow ? opn.a.bblk[NBIN] : 0, opt_.a.brow ? opt_.a.bblk[NBIN] : 0)),
                        ony);
        MPG_OPL(0);
        ++launches_per_iter;
        mark(mode == 0 ? PK_OP : PK_ASM);
      }
      if (need_p) {
        switch (Vop) {
          case 2: MPG_OPL(2); break;
          case 4: MPG_OPL(4); break;
          case 8: MPG_OPL(8); break;
          case 16: MPG_OPL(16); break;
          default: MPG_OPL(32); break;
        }
        ++launches_per_iter;
        mark(mode == 0 ? PK_OP : PK_ASM);
      }
    }
#undef MPG_OPL
    for (const Group& g : (mode == 0 ? op_groups_run : op_groups_asm)) {
      const OpView& ov = hs[size_t(g.idx[0])].transpose ? opt_ : opn;
      const unsigned gfull = cdiv(nb * int64_t(Vop), 256);
      const unsigned grid1 = mode == 0 ? gfull : std::min<unsigned>(gfull, unsigned(c.sm_count) * 8u);
#define MPG_OPM(VV)                                                                                            \
  switch (op.emode) {                                                                                          \
    case E_IDENT: k_iter_op_multi<VV, E_IDENT><<<grid1, 256, 0, s>>>(dS.get(), g, ov, mode); break;           \
    case E_DIAG: k_iter_op_multi<VV, E_DIAG><<<grid1, 256, 0, s>>>(dS.get(), g, ov, mode); break;             \
    default: k_iter_op_multi<VV, E_SAMEPAT><<<grid1, 256, 0, s>>>(dS.get(), g, ov, mode); break;              \
  }
      switch (Vop) {
        case 2: MPG_OPM(2); break;
        case 4: MPG_OPM(4); break;
        case 8: MPG_OPM(8); break;
        case 16: MPG_OPM(16); break;
        default: MPG_OPM(32); break;
      }
#undef MPG_OPM
      ++launches_per_iter;
      mark(mode == 0 ? PK_OP : PK_ASM);
    }
  };
  const dim3 gG{unsigned(G), unsigned(ns), 1u};
  const dim3 gR{cdiv(maxit + 2, 8), unsigned(ns), 1u};
  auto record_iteration = [&] {
    launches_per_iter = 0;
    for (int st = 0; st < max_stages; ++st) chain_stage(st, 0);
    iter_op(0);
    if (fused) {
      // projection: k_gs_tmx<true> for k + 2 <= GX_MAXV when the panel tensor maps exist
      // (MPG_GS_DOT=reg keeps the register-tiled kernel for every k)
      if (f32_on) {
        k_shadow<<<dim3(unsigned(std::min<int64_t>(cdiv(nmax, 1024), 1024)), unsigned(ns)), 256, 0, s>>>(dS.get(), psel);
        k_gs_tmxf<<<unsigned(gc_dot.ncl), GX_THREADS, GF_SMEM, s>>>(dS.get(), ns, G, psel);
        launches_per_iter += 2;
      } else if (psel.sel & 4) {
        k_gs_tmx<true><<<unsigned(gc_dot.ncl), GX_THREADS, GX_SMEM, s>>>(dS.get(), ns, G, psel);
        ++launches_per_iter;
      }
      MPG_CUDA(gc_launch_any(false, gc_dot, s, dS.get(), ns, G, psel));
    } else {
      k_dot<<<gG, 256, smem_dot, s>>>(dS.get(), G);
    }
    mark(PK_DOT);
    k_reduce<<<gR, 256, 0, s>>>(dS.get(), G, 0, fused ? gc_dot.ncl : G);
    mark(PK_SMALL);
    if (dcgs_on) {
      k_dcgs_fix<<<unsigned(ns), 256, 0, s>>>(dS.get());
      ++launches_per_iter;
      mark(PK_SMALL);
    }
    if (fused) {
      --launches_per_iter;
      // one profile interval for the pass, whichever kernels own its solves
      if (need_tma) {
        k_gs_tma<<<unsigned(gc_upd.ncl), GT_THREADS, GT_SMEM, s>>>(dS.get(), ns, G, usel);
        ++launches_per_iter;
      }
      if (need_tmx) {
        k_gs_tmx<false><<<unsigned(gc_upd.ncl), GX_THREADS, GX_SMEM, s>>>(dS.get(), ns, G, usel);
        ++launches_per_iter;
      }
      if (need_reg_upd) {
        MPG_CUDA(gc_launch_any(true, gc_upd, s, dS.get(), ns, G, usel));
        ++launches_per_iter;
      }
      mark(PK_UPDPROBE);
    } else {
      k_update<<<gG, 256, smem_upd, s>>>(dS.get(), G, 0);
      mark(PK_UPD);
      k_dot<<<gG, 256, smem_dot, s>>>(dS.get(), G);
      mark(PK_PROBE);
    }
    k_reduce<<<gR, 256, 0, s>>>(dS.get(), G, 1, fused ? gc_upd.ncl : G);
    mark(PK_SMALL);
    if (fused) {
      k_reorth_p<<<unsigned(c.sm_count), RO_THREADS, smem_ro, s>>>(dS.get(), ns, G, psel);
    } else {
      k_update<<<gG, 256, smem_upd, s>>>(dS.get(), G, 1);
    }
    mark(PK_REORTH);
    k_finalize<<<unsigned(ns), 32, 0, s>>>(dS.get(), G, fused ? c.sm_count : G, psel);
    mark(PK_SMALL);
    k_backsub<<<unsigned(ns), 256, size_t(maxit + 2) * sizeof(double), s>>>(dS.get());
    mark(PK_ASM);
    k_update<<<gG, 256, smem_upd, s>>>(dS.get(), G, 2);
    mark(PK_ASM);
    launches_per_iter += 9;
    for (int st = 0; st < max_stages; ++st) chain_stage(st, 1);
    iter_op(1);
    k_rnorm<<<gG, 256, 0, s>>>(dS.get(), G);
    mark(PK_ASM);
    k_post<<<unsigned(ns), 32, 0, s>>>(dS.get(), G);
    mark(PK_SMALL);
    launches_per_iter += 2;
  };
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const bool profiling = profile_enabled();
  if (!profiling) {
    MPG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    record_iteration();
    cudaError_t cap_err = cudaGetLastError();
    MPG_CUDA(cudaStreamEndCapture(s, &graph));
    if (cap_err != cudaSuccess) throw CudaError(std::string("gmres graph capture: ") + cudaGetErrorString(cap_err));
    MPG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  }
  // Profiled iteration: direct launches bracketed by events; algorithmic bytes
  // per kernel class from the per-solve state before the iteration.
  std::vector<cudaEvent_t> evs;
  std::vector<int> ev_kind;
  auto profiled_iteration = [&] {
    std::vector<GmSolve> before = hs;
    ev_kind.clear();
    auto take = [&](int kind) {
      if (evs.size() < ev_kind.size() + 2) {
        cudaEvent_t e;
        MPG_CUDA(cudaEventCreate(&e));
        evs.push_back(e);
      }
      ev_kind.push_back(kind);
      MPG_CUDA(cudaEventRecord(evs[ev_kind.size()], s));
    };
    if (evs.empty()) {
      cudaEvent_t e;
      MPG_CUDA(cudaEventCreate(&e));
      evs.push_back(e);
    }
    MPG_CUDA(cudaEventRecord(evs[0], s));
    mark = take;
    record_iteration();
    mark = [](int) {};
    MPG_CUDA(cudaMemcpyAsync(hs.data(), dS.get(), sizeof(GmSolve) * size_t(ns), cudaMemcpyDeviceToHost, s));
    MPG_CUDA(cudaStreamSynchronize(s));
    // Algorithmic bytes of the launches (4-byte indices, 8-byte values): a matrix
    // that one interleaved group kernel streams for all its solves is counted once
    // per group, the vectors per solve.
    double bytes[PK_COUNT] = {};
    std::vector<char> leader(size_t(ns), 1);
    for (size_t gi = 0; gi < chain_groups.size(); ++gi)
      if (chain_il[gi])
        for (int q = 1; q < il_groups[gi].cnt; ++q)
          if (il_groups[gi].idx[q] != il_groups[gi].idx[0]) leader[size_t(il_groups[gi].idx[q])] = 0;
    for (int i = 0; i < ns; ++i) {
      const GmSolve& b = before[size_t(i)];
      if (b.phase != PH_RUN) continue;
      const double n = double(b.n), k = double(b.k);
      const double lead = leader[size_t(i)] ? 1.0 : 0.0;
      for (int stg = 0; stg < b.stages; ++stg) {
        const DevCsr& f = *specs[size_t(i)].chain->factors[size_t(stg)];
        const double h = b.pair_bd ? 2.0 : 1.0;
        bytes[PK_CHAIN] += h * (lead * (12.0 * double(f.nnz) + 4.0 * double(f.nrows + 1)) + 16.0 * double(f.nrows));
      }
      const double vec = b.pair ? 2.0 : 1.0;
      const double be = op.emode == E_SAMEPAT ? 8.0 * double(op.a->nnz) : op.emode == E_DIAG ? 8.0 * double(nb) : 0.0;
      bytes[PK_OP] += lead * (12.0 * double(op.a->nnz) + 4.0 * double(nb + 1) + be) + vec * 16.0 * double(nb);
      const bool pf32 = b.F != nullptr && (psel.sel & 4) && b.tm != nullptr && b.k + 2 <= GX_MAXV && b.k + 1 > psel.split;
      if (pf32)  // float shadow of columns 0..k-1, w and V[k] in fp64, V[k]'s correction and shadow written
        bytes[PK_DOT] += 4.0 * n * k + 16.0 * n + (b.pend ? 8.0 * n : 0.0) + 4.0 * n;
      else
        bytes[PK_DOT] += 8.0 * n * (k + 1.0) + 8.0 * n + (b.pend ? 8.0 * n : 0.0) + (b.F ? 12.0 * n : 0.0);
      bytes[PK_UPDPROBE] += 8.0 * n * (k + 1.0) + 16.0 * n;
      bytes[PK_UPD] += 8.0 * n * (k + 1.0) + 16.0 * n;
      bytes[PK_PROBE] += 8.0 * n * (k + 1.0) + 8.0 * n;
      // an immediate second pass (a delayed one is folded into the next projection)
      if (hs[size_t(i)].reorth_count > b.reorth_count && !hs[size_t(i)].pend)
        bytes[PK_REORTH] += 8.0 * n * (k + 1.0) + 16.0 * n;
    }
    for (size_t e = 0; e < ev_kind.size(); ++e) {
      float ms = 0.0f;
      MPG_CUDA(cudaEventElapsedTime(&ms, evs[e], evs[e + 1]));
      profile_add(ev_kind[e], double(ms), 1);
    }
    for (int kk = 0; kk < PK_COUNT; ++kk)
      if (bytes[kk] > 0.0) profile_add_bytes(kk, bytes[kk]);
  };

  // ---- host loop: launch chunks, poll phases ----
  const double t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<int> khost(size_t(ns), 0);
  std::vector<double> done_at(size_t(ns), -1.0);
  int chunk = 4;
  try {
    while (true) {
      bool active = false;
      for (int i = 0; i < ns; ++i)
        if (hs[size_t(i)].phase != PH_DONE) {
          active = true;
          ensure(i, khost[size_t(i)] + chunk + 2);
        }
      if (!active) break;
      if (profiling) {
        for (int t = 0; t < chunk; ++t) profiled_iteration();
      } else {
        for (int t = 0; t < chunk; ++t) MPG_CUDA(cudaGraphLaunch(exec, s));
      }
      count_launch(int64_t(chunk) * launches_per_iter);
      MPG_CUDA(cudaMemcpyAsync(hs.data(), dS.get(), sizeof(GmSolve) * size_t(ns), cudaMemcpyDeviceToHost, s));
      MPG_CUDA(cudaStreamSynchronize(s));
      const double now = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      for (int i = 0; i < ns; ++i) {
        khost[size_t(i)] = hs[size_t(i)].k;
        if (hs[size_t(i)].phase == PH_DONE && done_at[size_t(i)] < 0) done_at[size_t(i)] = now;
      }
      chunk = std::min(chunk * 2, 32);
    }
  } catch (...) {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto e : evs) cudaEventDestroy(e);
    throw;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  for (auto e : evs) cudaEventDestroy(e);
  if (std::getenv("MPG_GMRES_TIMING")) {
    int maxk = 0;
    for (const auto& g : hs) maxk = std::max(maxk, g.iterations);
    std::fprintf(stderr, "gmres_batch: %d solves, setup %.3f s, total %.3f s, max its %d\n", ns, t_setup,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), maxk);
  }

  // ---- outputs ----
  for (int i = 0; i < ns; ++i) {
    const GmSolve& g = hs[size_t(i)];
    SolveHost& H = sh[size_t(i)];
    GmresOutcome& o = out[size_t(i)];
    o.iterations = g.iterations;
    o.converged = g.converged;
    o.breakdown = g.breakdown;
    o.rhs_norm = g.bnorm;
    o.final_residual = g.final_residual;
    o.solve_seconds = done_at[size_t(i)];
    o.reorth_passes = g.reorth_count;
    if (opt.record_history) {
      o.history.resize(size_t(g.iterations) + 1);
      MPG_CUDA(cudaMemcpyAsync(o.history.data(), H.hist.get(), o.history.size() * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
    }
    if (specs[size_t(i)].x) {
      const double* src = g.xsel == 0 ? H.ubuf.get() : g.xsel == 1 ? H.z0.get() : g.xsel == 2 ? H.z1.get() : nullptr;
      if (src) {
        copy_out(specs[size_t(i)].x, src, size_t(g.n), s);
      } else if (is_device_ptr(specs[size_t(i)].x)) {
        MPG_CUDA(cudaMemsetAsync(specs[size_t(i)].x, 0, size_t(g.n) * sizeof(double), s));
      } else {
        MPG_CUDA(cudaStreamSynchronize(s));
        std::memset(specs[size_t(i)].x, 0, size_t(g.n) * sizeof(double));
      }
    }
  }
  MPG_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace mpg
