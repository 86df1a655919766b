// Read-bandwidth ceilings of the Gram-Schmidt access patterns on B200
// (tuning aid, not part of the library). V = nv vectors of ld doubles, flat.
//   tile:   one CTA per SM, 512 threads, tiles of T rows x nv vectors, thread
//           (rg, cg) loads CPT double2 per tile, register double buffer
//   rowthr: k_update pattern: thread owns 2 rows, loops over the nv vectors
//   colstr: warp streams one vector over a contiguous chunk of R rows
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_sink(double v, double* out) { if (v == 12345.678) out[0] = v; }

template <int RG, int CPT>
__global__ void __launch_bounds__(512, 1) k_tile(const double* __restrict__ V, int nv, int ld, int n, double* out, int blocked) {
  constexpr int CG = 512 / RG, T = 2 * RG;
  const int rg = threadIdx.x % RG, cg = threadIdx.x / RG;
  const int ncol = nv > cg ? min(CPT, (nv - cg + CG - 1) / CG) : 0;
  const int ntl = (n + T - 1) / T, per = (ntl + gridDim.x - 1) / gridDim.x;
  const int t0 = blocked ? blockIdx.x * per : blockIdx.x, t1 = blocked ? min(ntl, t0 + per) : ntl, ts = blocked ? 1 : gridDim.x;
  double acc = 0.0;
  double2 a[CPT], b[CPT];
  auto load = [&](int t, double2* v) {
#pragma unroll
    for (int c = 0; c < CPT; ++c)
      v[c] = (c < ncol && t < t1) ? __ldcs(reinterpret_cast<const double2*>(V + size_t(cg + CG * c) * ld + t * T + 2 * rg))
                                  : make_double2(0, 0);
  };
  auto use = [&](const double2* v) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc += v[c].x * 1.0000001 + v[c].y;
  };
  int t = t0;
  load(t, a);
  while (t < t1) {
    load(t + ts, b);
    use(a);
    t += ts;
    if (t >= t1) break;
    load(t + ts, a);
    use(b);
    t += ts;
  }
  if (acc == 12345.678) out[0] = acc;
}

// Same walk on a chunk-major layout [n / T][nv][T]: the tile of every vector is
// one contiguous nv x T x 8-byte block.
template <int RG, int CPT>
__global__ void __launch_bounds__(512, 1) k_tile_cm(const double* __restrict__ V, int nv, int ld, int n, double* out) {
  constexpr int CG = 512 / RG, T = 2 * RG;
  const int rg = threadIdx.x % RG, cg = threadIdx.x / RG;
  const int ncol = nv > cg ? min(CPT, (nv - cg + CG - 1) / CG) : 0;
  const int ntl = (n + T - 1) / T;
  double acc = 0.0;
  double2 a[CPT], b[CPT];
  auto load = [&](int t, double2* v) {
#pragma unroll
    for (int c = 0; c < CPT; ++c)
      v[c] = (c < ncol && t < ntl) ? __ldcs(reinterpret_cast<const double2*>(V + (size_t(t) * nv + cg + CG * c) * T + 2 * rg))
                                   : make_double2(0, 0);
  };
  auto use = [&](const double2* v) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc += v[c].x * 1.0000001 + v[c].y;
  };
  int t = blockIdx.x;
  load(t, a);
  while (t < ntl) {
    load(t + gridDim.x, b);
    use(a);
    t += gridDim.x;
    if (t >= ntl) break;
    load(t + gridDim.x, a);
    use(b);
    t += gridDim.x;
  }
  if (acc == 12345.678) out[0] = acc;
}

// CTA pairs (cluster of 2) walking adjacent T-row tiles in lockstep: a relaxed
// cluster barrier per tile keeps the two SMs' requests to neighbouring
// segments of each vector together in time (no data exchanged).
template <int RG, int CPT, int SYNC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    k_tile_pair(const double* __restrict__ V, int nv, int ld, int n, double* out) {
  constexpr int CG = 512 / RG, T = 2 * RG;
  const int rg = threadIdx.x % RG, cg = threadIdx.x / RG;
  const int q = blockIdx.x & 1, pr = blockIdx.x >> 1, npr = gridDim.x >> 1;
  const int ncol = nv > cg ? min(CPT, (nv - cg + CG - 1) / CG) : 0;
  const int nst = (n + 2 * T - 1) / (2 * T);
  double acc = 0.0;
  double2 a[CPT], b[CPT];
  auto load = [&](int st, double2* v) {
    const int row = st * 2 * T + q * T + 2 * rg;
#pragma unroll
    for (int c = 0; c < CPT; ++c)
      v[c] = (c < ncol && st < nst && row < ld) ? __ldcs(reinterpret_cast<const double2*>(V + size_t(cg + CG * c) * ld + row))
                                               : make_double2(0, 0);
  };
  auto use = [&](const double2* v) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc += v[c].x * 1.0000001 + v[c].y;
    if (SYNC) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    }
  };
  int st = pr;
  load(st, a);
  while (st < nst) {  // same trip count in both CTAs of the pair
    load(st + npr, b);
    use(a);
    st += npr;
    if (st >= nst) break;
    load(st + npr, a);
    use(b);
    st += npr;
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) k_rowthr(const double* __restrict__ V, int nv, int ld, int n, double* out) {
  const int r = 2 * (blockIdx.x * 256 + threadIdx.x);
  if (r >= n) return;
  double2 acc = make_double2(0, 0);
  int j = 0;
  for (; j + U <= nv; j += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(V + size_t(j + u) * ld + r));
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += 1.0000001 * v[u].x; acc.y += v[u].y; }
  }
  for (; j < nv; ++j) { double2 v = __ldcs(reinterpret_cast<const double2*>(V + size_t(j) * ld + r)); acc.x += v.x; acc.y += v.y; }
  if (acc.x + acc.y == 12345.678) out[0] = acc.x;
}

template <int U>
__global__ void __launch_bounds__(512) k_colstr(const double* __restrict__ V, int nv, int ld, int n, int R, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (n + R - 1) / R;
  double acc = 0.0;
  for (int ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int r0 = ch * R, r1 = min(n, r0 + R);
    for (int j = warp; j < nv; j += 16) {
      const double* v = V + size_t(j) * ld;
      for (int r = r0 + 2 * lane; r < r1; r += 64 * U) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int rr = r + 64 * u;
          x[u] = rr < r1 ? __ldcs(reinterpret_cast<const double2*>(v + rr)) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += 1.0000001 * x[u].x + x[u].y;
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1191016;
  const int nv = argc > 2 ? atoi(argv[2]) : 300;
  const int ld = (n + 31) / 32 * 32;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *V, *out;
  CK(cudaMalloc(&V, size_t(nv) * ld * 8));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(V, 0, size_t(nv) * ld * 8));
  // flush buffer larger than L2
  double* fl;
  const size_t flb = size_t(512) << 20;
  CK(cudaMalloc(&fl, flb));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = double(nv) * n * 8;
  auto timeit = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemsetAsync(fl, rep, flb));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-40s %8.3f ms %8.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  char nm[128];
#define TILE(RG, CPT, BL)                                                                               \
  cudaFuncSetAttribute(k_tile<RG, CPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);               \
  snprintf(nm, sizeof nm, "tile RG=%d CPT=%d blocked=%d", RG, CPT, BL);                               \
  timeit(nm, [&] { k_tile<RG, CPT><<<sms, 512>>>(V, nv, ld, n, out, BL); });
  if (nv <= 512 / 8 * 8) { TILE(8, 8, 0); TILE(8, 8, 1); }
  if (nv <= 512 / 4 * 8 && nv > 256) { TILE(4, 8, 0); }
  if (nv <= 512 / 16 * 8) { TILE(16, 8, 0); }
  if (nv <= 512 / 8 * 4) { TILE(8, 4, 0); }
  if (nv <= 512 / 4 * 4) { TILE(4, 4, 0); }
  if (nv <= 512 / 4 * 16) { TILE(4, 16, 0); }
  if (nv <= 512 / 2 * 8) { TILE(2, 8, 0); }
  if (nv <= 512) {
    snprintf(nm, sizeof nm, "chunk-major RG=8 CPT=8");
    timeit(nm, [&] { k_tile_cm<8, 8><<<sms, 512>>>(V, nv, ld, n, out); });
    snprintf(nm, sizeof nm, "chunk-major RG=4 CPT=8");
    timeit(nm, [&] { k_tile_cm<4, 8><<<sms, 512>>>(V, nv, ld, n, out); });
  }
  snprintf(nm, sizeof nm, "pair RG=8 CPT=8 sync=1");
  timeit(nm, [&] { k_tile_pair<8, 8, 1><<<sms / 2 * 2, 512>>>(V, nv, ld, n, out); });
  snprintf(nm, sizeof nm, "pair RG=8 CPT=8 sync=0");
  timeit(nm, [&] { k_tile_pair<8, 8, 0><<<sms / 2 * 2, 512>>>(V, nv, ld, n, out); });
  snprintf(nm, sizeof nm, "rowthr U=4");
  timeit(nm, [&] { k_rowthr<4><<<(n / 2 + 255) / 256, 256>>>(V, nv, ld, n, out); });
  snprintf(nm, sizeof nm, "rowthr U=8");
  timeit(nm, [&] { k_rowthr<8><<<(n / 2 + 255) / 256, 256>>>(V, nv, ld, n, out); });
  for (int R : {2048, 8192, 32768}) {
    for (int g : {sms, 2 * sms, 4 * sms}) {
      snprintf(nm, sizeof nm, "colstr U=4 R=%d grid=%d", R, g);
      timeit(nm, [&] { k_colstr<4><<<g, 512>>>(V, nv, ld, n, R, out); });
      snprintf(nm, sizeof nm, "colstr U=8 R=%d grid=%d", R, g);
      timeit(nm, [&] { k_colstr<8><<<g, 512>>>(V, nv, ld, n, R, out); });
    }
  }
  return 0;
}
