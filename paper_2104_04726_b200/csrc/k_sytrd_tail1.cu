// Single-CTA tail of the Householder tridiagonalisation (dsytrd's role in eigh,
// tensor.py:195).
//
// Once the trailing block is small, the grid-wide kernel (k_sytrd_smem) spends
// its ~6k cycles per column on latency -- a 148-block grid barrier (~2.5k
// cycles, the measured floor on B200), two block reductions and an L2 gather
// -- for a few hundred cycles of work. Here ONE 1024-thread CTA holds the whole
// trailing m x m block (m <= T1_MAX) in shared memory and runs the same
// algorithm with two block barriers per column: the Householder scalars in
// warp 0 (registers, shuffles), then one fused pass in which thread (row i,
// column stride s) applies the rank-2 update of step k and accumulates row i
// of p_{k+1} = T' v_{k+1} (T symmetric, so no cross-thread reduction beyond 4
// partials). It continues from step K0 exactly where the
// grid kernel stopped: v_{K0} in hv column K0, tau_{K0} in tau, the trailing
// block (rows/columns >= K0+1) of A updated through step K0-1.
// Deterministic: fixed reduction trees.
#include <cstdio>
#include <cstdlib>

#include "tmb_internal.cuh"

namespace tmb {
namespace {

constexpr int T1_THREADS = 1024;
constexpr int T1_WARPS = T1_THREADS / 32;

__device__ __forceinline__ double wsum1(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double frcp1(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}

constexpr int T1_MAX = 160;                     // trailing block capacity (227 KB of shared memory)
constexpr int T1_RPL = (T1_MAX + 31) / 32;      // live rows per lane of warp 0
#ifndef TMB_T1_PARTS
#define TMB_T1_PARTS 4
#endif
constexpr int T1_PARTS = TMB_T1_PARTS;          // symv: T1_THREADS / T1_PARTS rows x T1_PARTS column strides
constexpr int T1_ROWS = T1_THREADS / T1_PARTS;

__global__ void __launch_bounds__(T1_THREADS, 1) k_sytrd_tail1(double* __restrict__ A, int64_t n, int64_t K0,
                                                              double* __restrict__ d, double* __restrict__ e,
                                                              double* __restrict__ tau, double* __restrict__ hv,
                                                              long long* __restrict__ prof) {
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;  // TMB_TRD_PROFILE: per-phase cycles summed over the columns
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = K0 + 1;
  const int m = (int)(n - base);
  extern __shared__ double sm[];
  double* T = sm;                  // m x m, column-major, ld m: trailing block (local index = global - base)
  double* v = T + m * m;           // m: v_k
  double* w = v + m;               // m: w_k
  double* x = w + m;               // m: v_{k+1}
  double* pp = x + m;              // T1_PARTS x m: partial sums of p = T v (row i, column stride part)
  double* sc = pp + T1_PARTS * m;  // [1] tau_{k+1}
  for (int lj = warp; lj < m; lj += T1_WARPS)
    for (int li = lane; li < m; li += 32) T[li + m * lj] = A[(base + li) + n * (base + lj)];
  for (int li = tid; li < m; li += T1_THREADS) v[li] = hv[(base + li) + n * K0];
  double tau_k = tau[K0];
  __syncthreads();
  const int srow = tid % T1_ROWS, spart = tid / T1_ROWS;
  for (int li = srow; li < m; li += T1_ROWS) {  // p_{K0} partials (no update pending)
    double acc = 0.0;
    for (int lj = spart; lj < m; lj += T1_PARTS) acc = fma(T[li + m * lj], v[lj], acc);
    pp[spart * m + li] = acc;
  }
  __syncthreads();

  for (int64_t k = K0; k + 2 < n; ++k) {
    if (prof && threadIdx.x == 0) t0 = clock64();
    const int r0 = (int)(k + 1 - base);  // local index of column k+1
    if (warp == 0) {
      // lane owns live rows li = r0 + lane + 32 q; the scalar chain stays in registers
      double vr[T1_RPL], wr[T1_RPL], xr[T1_RPL];
      double pv = 0.0;
#pragma unroll
      for (int q = 0; q < T1_RPL; ++q) {
        const int li = r0 + lane + 32 * q;
        vr[q] = wr[q] = xr[q] = 0.0;
        if (li < m) {
          double p = pp[li];
#pragma unroll
          for (int pt = 1; pt < T1_PARTS; ++pt) p += pp[pt * m + li];
          vr[q] = v[li];
          wr[q] = tau_k * p;
          xr[q] = T[li + m * r0];
          pv = fma(wr[q], vr[q], pv);
        }
      }
      const double K = 0.5 * tau_k * wsum1(pv);
#pragma unroll
      for (int q = 0; q < T1_RPL; ++q) wr[q] = wr[q] - K * vr[q];  // w_k = p - K v
      const double w_c1 = __shfl_sync(0xffffffffu, wr[0], 0), v_c1 = __shfl_sync(0xffffffffu, vr[0], 0);
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < T1_RPL; ++q) {
        const int li = r0 + lane + 32 * q;
        if (li < m) {
          xr[q] = xr[q] - vr[q] * w_c1 - wr[q] * v_c1;
          w[li] = wr[q];
          if (li >= r0 + 2) s2 = fma(xr[q], xr[q], s2);
        }
      }
      s2 = wsum1(s2);
      if (k + 3 == n) {  // last 2x2 block: finish d/e directly
        const double x0 = __shfl_sync(0xffffffffu, xr[0], 0), x1 = __shfl_sync(0xffffffffu, xr[0], 1);
        const double vl = __shfl_sync(0xffffffffu, vr[0], 1), wl = __shfl_sync(0xffffffffu, wr[0], 1);
        if (lane == 0) {
          d[n - 2] = x0;
          e[n - 2] = x1;
          d[n - 1] = T[(m - 1) + m * (m - 1)] - 2.0 * vl * wl;
          tau[n - 2] = 0.0;
        }
      } else {
        const double alpha = __shfl_sync(0xffffffffu, xr[0], 1), xc1 = __shfl_sync(0xffffffffu, xr[0], 0);
        double tau_n = 0.0, beta = alpha, scale = 0.0;
        if (s2 > 0.0) {
          const double nrm = sqrt(alpha * alpha + s2);
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau_n = (beta - alpha) * frcp1(beta);
          scale = frcp1(alpha - beta);
        }
        if (lane == 0) {
          d[k + 1] = xc1;
          e[k + 1] = beta;
          tau[k + 1] = tau_n;
          sc[1] = tau_n;
        }
#pragma unroll
        for (int q = 0; q < T1_RPL; ++q) {
          const int li = r0 + lane + 32 * q;
          if (li < m) x[li] = li == r0 + 1 ? 1.0 : (li >= r0 + 2 ? xr[q] * scale : 0.0);
        }
      }
    }
    __syncthreads();
    if (prof && threadIdx.x == 0) t1 = clock64();
    if (k + 3 == n) break;
    // reflector k+1 into hv (full column, zero above row k+2)
    {
      double* h = hv + n * (k + 1);
      for (int64_t i = tid; i < n; i += T1_THREADS) h[i] = (i >= base && i - base > r0) ? x[i - base] : 0.0;
    }
    // fused pass over the block that stays live (rows/columns >= r0+1): rank-2
    // update of step k and, through the symmetry of T, the row sums of p_{k+1}
    for (int li = r0 + 1 + srow; li < m; li += T1_ROWS) {
      const int r1 = r0 + 1;
      {
        const double vi = v[li], wi = w[li];
        double acc = 0.0;
#pragma unroll 4
        for (int lj = r1 + spart; lj < m; lj += T1_PARTS) {
          double* t = T + li + m * lj;
          const double tv = *t - vi * w[lj] - wi * v[lj];
          *t = tv;
          acc = fma(tv, x[lj], acc);
        }
        pp[spart * m + li] = acc;
      }
    }
    tau_k = sc[1];
    __syncthreads();
    if (prof && threadIdx.x == 0) t2 = clock64();
    for (int li = r0 + 1 + tid; li < m; li += T1_THREADS) v[li] = x[li];
    __syncthreads();
    if (prof && threadIdx.x == 0) {
      t3 = clock64();
      prof[0] += t1 - t0; prof[1] += t2 - t1; prof[2] += t3 - t2; prof[3] += 1;
    }
  }
}

}  // namespace

int64_t sytrd_tail1_max() {
  static const int64_t env = [] {
    const char* s = std::getenv("TMB_SYTRD_TAIL1");  // A/B: trailing size handed to the single-CTA kernel (0 = off)
    return s ? std::atoll(s) : (int64_t)-1;
  }();
  // measured (bench_eig.py, C2 sizes): trailing 96-128 best (n=1080 4.26 vs 4.37 ms without the
  // tail kernel, n=1920 8.56 vs 8.65); 160 gives back part of it (the block pass grows as m^2)
  return env >= 0 ? std::min<int64_t>(env, T1_MAX) : 128;
}

void sytrd_tail1(Ctx& c, double* A, int64_t n, int64_t K0, double* d, double* e, double* tau, double* hv) {
  const int64_t m = n - K0 - 1;
  if (m < 2 || m > T1_MAX) throw Error(TMB_EINVAL, "sytrd_tail1: trailing block size out of range");
  const size_t smem = sizeof(double) * ((size_t)m * m + (3 + T1_PARTS) * (size_t)m + 2);
  set_smem_attr(c, (const void*)k_sytrd_tail1, sizeof(double) * (T1_MAX * T1_MAX + (3 + T1_PARTS) * T1_MAX + 2));
  static const bool prof_on = std::getenv("TMB_TRD_PROFILE") != nullptr;
  long long* prof = nullptr;
  if (prof_on) {
    prof = alloc<long long>(c, 4);
    TMB_CUDA(cudaMemsetAsync(prof, 0, 4 * sizeof(long long), c.stream));
  }
  k_sytrd_tail1<<<1, T1_THREADS, smem, c.stream>>>(A, n, K0, d, e, tau, hv, prof);
  c.launches++;
  check_launch("k_sytrd_tail1");
  if (prof) {
    long long h[4];
    TMB_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    if (h[3])
      std::fprintf(stderr, "sytrd_tail1 n=%lld m=%lld cycles/column: scalars+bar %lld | hv+pass+bar %lld | copy+bar %lld\n",
                   (long long)n, (long long)m, h[0] / h[3], h[1] / h[3], h[2] / h[3]);
  }
}

}  // namespace tmb
