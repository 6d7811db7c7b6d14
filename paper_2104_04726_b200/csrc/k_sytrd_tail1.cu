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
constexpr int T1_PARTS_MAX = 16;

// T1_THREADS threads; symv: T1_THREADS / T1_PARTS rows x T1_PARTS column strides
template <int T1_THREADS, int T1_PARTS>
__global__ void __launch_bounds__(T1_THREADS, 1) k_sytrd_tail1(double* __restrict__ A, int64_t n, int64_t K0,
                                                              double* __restrict__ d, double* __restrict__ e,
                                                              double* __restrict__ tau, double* __restrict__ hv,
                                                              long long* __restrict__ prof) {
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;  // TMB_TRD_PROFILE: per-phase cycles summed over the columns
  constexpr int T1_WARPS = T1_THREADS / 32;
  constexpr int T1_ROWS = T1_THREADS / T1_PARTS;
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

// Register-tiled variant (m <= 128): the trailing block lives in REGISTERS. 256 threads;
// warp w owns rows [16 w, 16 w + 16), lane l columns [4 l, 4 l + 4): a 16 x 4 tile per thread.
// A warp covers all columns of its rows, so the row sums of p_{k+1} = T' v_{k+1} need only a
// warp reduce-scatter (no cross-warp partials), and the fused pass touches shared memory only
// for the vectors (v_k, w_k interleaved, v_{k+1}): ~1 load per 3 elements instead of 5 per
// element in the shared-memory-matrix kernel above. Per column: the Householder scalars in
// warp 0 (as above), one barrier, the pass, one barrier. Dead rows/columns of a tile keep
// being updated with finite garbage that nothing reads (v_{k+1} is zero there).
constexpr int T2_M = 128, T2_THREADS = 256, T2_RPL = T2_M / 32;

__global__ void __launch_bounds__(T2_THREADS, 1) k_sytrd_tail2(double* __restrict__ A, int64_t n, int64_t K0,
                                                              double* __restrict__ d, double* __restrict__ e,
                                                              double* __restrict__ tau, double* __restrict__ hv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = K0 + 1;
  const int m = (int)(n - base);
  __shared__ __align__(16) double2 vw[T2_M];      // (v_k, w_k)
  __shared__ __align__(16) double xb[2][T2_M];    // v_{k+1} (double-buffered: it is v_k of the next step)
  __shared__ double xcol[T2_M];                   // the next pivot column, published by the pass
  __shared__ double pr[T2_M];                     // row sums of T v (unscaled)
  __shared__ double sc[2];                        // [0] tau_{k+1}, [1] T[m-1][m-1]
  const int i0 = 16 * warp, j0 = 4 * lane;
  double t[16][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int i = i0 + r, j = j0 + c;
      t[r][c] = (i < m && j < m) ? A[(base + i) + n * (base + j)] : 0.0;
      if (i == m - 1 && j == m - 1) sc[1] = t[r][c];
    }
  for (int li = tid; li < T2_M; li += T2_THREADS) {
    xb[0][li] = li < m ? hv[(base + li) + n * K0] : 0.0;
    xb[1][li] = 0.0;
    vw[li] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  // p_{K0} = T v_{K0} row sums (no update pending) and the first pivot column (local 0)
  {
    double xc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) xc[c] = xb[0][j0 + c];
    double acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      acc[r] = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r] = fma(t[r][c], xc[c], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double s = wsum1(acc[r]);
      if (lane == 0) pr[i0 + r] = s;
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < 16; ++r) xcol[i0 + r] = t[r][0];
    }
  }
  __syncthreads();
  double tau_k = tau[K0];
  int cur = 0;  // xb[cur] = v_k
  for (int64_t k = K0; k + 2 < n; ++k) {
    const int r0 = (int)(k + 1 - base);  // local index of column k+1
    const double* vk = xb[cur];
    double* xn = xb[cur ^ 1];
    if (warp == 0) {
      double vr[T2_RPL], wr[T2_RPL], xr[T2_RPL];
      double pv = 0.0;
#pragma unroll
      for (int q = 0; q < T2_RPL; ++q) {
        const int li = r0 + lane + 32 * q;
        vr[q] = wr[q] = xr[q] = 0.0;
        if (li < m) {
          vr[q] = vk[li];
          wr[q] = tau_k * pr[li];
          xr[q] = xcol[li];
          pv = fma(wr[q], vr[q], pv);
        }
      }
      const double K = 0.5 * tau_k * wsum1(pv);
#pragma unroll
      for (int q = 0; q < T2_RPL; ++q) wr[q] = wr[q] - K * vr[q];  // w_k = p - K v
      const double w_c1 = __shfl_sync(0xffffffffu, wr[0], 0), v_c1 = __shfl_sync(0xffffffffu, vr[0], 0);
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < T2_RPL; ++q) {
        const int li = r0 + lane + 32 * q;
        if (li < m) {
          xr[q] = xr[q] - vr[q] * w_c1 - wr[q] * v_c1;
          vw[li] = make_double2(vr[q], wr[q]);
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
          d[n - 1] = sc[1] - 2.0 * vl * wl;
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
          sc[0] = tau_n;
        }
#pragma unroll
        for (int q = 0; q < T2_RPL; ++q) {
          const int li = r0 + lane + 32 * q;
          if (li < m) xn[li] = li == r0 + 1 ? 1.0 : (li >= r0 + 2 ? xr[q] * scale : 0.0);
        }
        // v_{k+1} is zero at and above the old pivot row; this buffer last held v_{k-1},
        // whose unit entry sits at r0 - 1
        if (lane == 0) xn[r0] = 0.0;
        if (lane == 1 && r0 >= 1) xn[r0 - 1] = 0.0;
      }
    }
    __syncthreads();
    if (k + 3 == n) break;
    // reflector k+1 into hv: rows >= base (the rows above were zeroed by the launcher)
    if (tid < m) hv[n * (k + 1) + base + tid] = tid > r0 ? xn[tid] : 0.0;
    const int r1 = r0 + 1;  // rows/columns >= r1 stay live
    if (i0 + 15 >= r1) {
      double vc[4], wc[4], xc[4];
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        const double2 a0 = vw[j0 + c], a1 = vw[j0 + c + 1];
        vc[c] = a0.x; wc[c] = a0.y; vc[c + 1] = a1.x; wc[c + 1] = a1.y;
        const double2 xx = *reinterpret_cast<const double2*>(xn + j0 + c);
        xc[c] = xx.x; xc[c + 1] = xx.y;
      }
      double acc[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        // no per-row branch (it would split the 16 independent rows into 16 dependent
        // basic blocks): rows of this warp that are already dead are updated with their
        // stale (finite) v, w and their sums are never read
        acc[r] = 0.0;
        const double2 rw = vw[i0 + r];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double tv = t[r][c] - rw.x * wc[c] - rw.y * vc[c];
          t[r][c] = tv;
          acc[r] = fma(tv, xc[c], acc[r]);
        }
      }
      // reduce-scatter of the 16 row sums over the 32 lanes (16 + 8 + 4 + 2 + 1 shuffles... as
      // halving exchanges: 8, 4, 2, 1, then one plain butterfly level)
      {
        const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
        double s8[8], s4[4], s2v[2];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          s8[i] = (b16 ? acc[8 + i] : acc[i]) + __shfl_xor_sync(0xffffffffu, b16 ? acc[i] : acc[8 + i], 16);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          s4[i] = (b8 ? s8[4 + i] : s8[i]) + __shfl_xor_sync(0xffffffffu, b8 ? s8[i] : s8[4 + i], 8);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          s2v[i] = (b4 ? s4[2 + i] : s4[i]) + __shfl_xor_sync(0xffffffffu, b4 ? s4[i] : s4[2 + i], 4);
        double s1 = (b2 ? s2v[1] : s2v[0]) + __shfl_xor_sync(0xffffffffu, b2 ? s2v[0] : s2v[1], 2);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        const int row = (b16 ? 8 : 0) + (b8 ? 4 : 0) + (b4 ? 2 : 0) + (b2 ? 1 : 0);
        if ((lane & 1) == 0) pr[i0 + row] = s1;
      }
      // the next pivot column (local r1) and, before the last step, the last diagonal element
      if (lane == (r1 >> 2)) {
        const int c1 = r1 & 3;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          double xv = t[r][0];
#pragma unroll
          for (int c = 1; c < 4; ++c) xv = c1 == c ? t[r][c] : xv;
          xcol[i0 + r] = xv;
        }
      }
      if (k + 4 == n && warp == ((m - 1) >> 4) && lane == ((m - 1) >> 2)) {
        const int rl = (m - 1) & 15, cl = (m - 1) & 3;
        double xv = 0.0;
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) xv = (rl == r && cl == c) ? t[r][c] : xv;
        sc[1] = xv;
      }
    }
    tau_k = sc[0];
    cur ^= 1;
    __syncthreads();
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
  // measured (scripts/gpu_s5_tail.sh): threads x column strides of the fused pass
  static const int shape_env = [] {
    // A/B: 0 = 1024 x 4, 1 = 1024 x 8, 2 = 512 x 4, 3 = 512 x 8, 4 = 256 x 4, 5 = 1024 x 16 (shared-memory
    // matrix), 9 = the register-tiled kernel for m <= 128 (else 512 x 4). Measured sytrd ms at n = 1080 /
    // 1920 (scripts/gpu_s5_tail.sh): 3.57 / 8.01, 3.58 / 8.02, 3.52 / 7.96, 3.53 / 7.96, 3.55 / 7.99,
    // 3.60 / 8.04; register-tiled 3.50 / 7.92 (the tail alone 289 -> 250 us)
    const char* s = std::getenv("TMB_T1_SHAPE");
    return s ? std::atoi(s) : 9;
  }();
  if (shape_env == 9 && m <= T2_M) {
    // rows above the trailing block of the tail's reflector columns: zero (one strided memset
    // instead of n stores per column on the kernel's serial path)
    if (m > 2)
      TMB_CUDA(cudaMemset2DAsync(hv + n * (K0 + 1), sizeof(double) * n, 0, sizeof(double) * (K0 + 1), (size_t)(m - 2),
                                 c.stream));
    k_sytrd_tail2<<<1, T2_THREADS, 0, c.stream>>>(A, n, K0, d, e, tau, hv);
    c.launches++;
    check_launch("k_sytrd_tail2");
    return;
  }
  using KFn = void (*)(double*, int64_t, int64_t, double*, double*, double*, double*, long long*);
  KFn kern;
  int nt, parts;
  switch (shape_env) {
    case 1: kern = k_sytrd_tail1<1024, 8>; nt = 1024; parts = 8; break;
    case 2: kern = k_sytrd_tail1<512, 4>; nt = 512; parts = 4; break;
    case 3: kern = k_sytrd_tail1<512, 8>; nt = 512; parts = 8; break;
    case 4: kern = k_sytrd_tail1<256, 4>; nt = 256; parts = 4; break;
    case 5: kern = k_sytrd_tail1<1024, 16>; nt = 1024; parts = 16; break;
    case 0: kern = k_sytrd_tail1<1024, 4>; nt = 1024; parts = 4; break;
    default: kern = k_sytrd_tail1<512, 4>; nt = 512; parts = 4; break;
  }
  const size_t smem = sizeof(double) * ((size_t)m * m + (3 + parts) * (size_t)m + 2);
  set_smem_attr(c, (const void*)kern, sizeof(double) * (T1_MAX * T1_MAX + (3 + T1_PARTS_MAX) * T1_MAX + 2));
  static const bool prof_on = std::getenv("TMB_TRD_PROFILE") != nullptr;
  long long* prof = nullptr;
  if (prof_on) {
    prof = alloc<long long>(c, 4);
    TMB_CUDA(cudaMemsetAsync(prof, 0, 4 * sizeof(long long), c.stream));
  }
  kern<<<1, nt, smem, c.stream>>>(A, n, K0, d, e, tau, hv, prof);
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
