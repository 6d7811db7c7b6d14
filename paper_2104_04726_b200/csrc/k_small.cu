// Memory-bound kernels: small-mode TTM / Gram (the colour and view-exposure
// modes, dims 3..64), deterministic fp64 reductions (fro_norm, tensor.py:212;
// fit, tucker.py:174-191; max factor change, tucker.py:319-323), the core
// quantiser (codec.py:98-99,114-134) and the sign rule (tensor.py:203-209).
// All reductions use a fixed grid and a fixed combination order, so results
// are bit-reproducible run to run.
#include "tmb_internal.cuh"

namespace tmb {
namespace {

constexpr int RED_BLOCKS = 1024;  // fixed => deterministic partial layout

template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t i) { return (double)p[i]; }

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;  // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, sh[i]);
  return s;
}

// ---- small-mode TTM: y[l + L(i + r rr)] = sum_k M(i,k) x[l + L(k + K rr)]
template <typename T>
__global__ void k_small_ttm(const T* __restrict__ x, int64_t L, int K, int64_t Rr,
                            const double* __restrict__ m, int r, int64_t sMr, int64_t sMk,
                            double* __restrict__ y) {
  extern __shared__ double sM[];  // [k][i]
  for (int e = threadIdx.x; e < K * r; e += blockDim.x) {
    const int k = e / r, i = e % r;
    sM[e] = m[i * sMr + k * sMk];
  }
  __syncthreads();
  const int nch = (r + 7) / 8;
  const int64_t total = L * Rr * nch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e % L, q = e / L;
    const int ich = (int)(q % nch);
    const int64_t rr = q / nch;
    double acc[8];
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) acc[ii] = 0.0;
    const T* xp = x + l + L * K * rr;
    for (int k = 0; k < K; ++k) {
      const double xv = ld(xp, L * k);
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        const int i = ich * 8 + ii;
        if (i < r) acc[ii] = fma(sM[k * r + i], xv, acc[ii]);
      }
    }
    double* yp = y + l + L * r * rr;
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) {
      const int i = ich * 8 + ii;
      if (i < r) yp[L * i] = acc[ii];
    }
  }
}

// ---- two consecutive small-mode TTMs in one pass (modes m, m+1 both small):
// y[l + L(i1 + r1 (i2 + r2 rr))] = sum_k2 M2(i2,k2) sum_k1 M1(i1,k1) x[l + L(k1 + K1 (k2 + K2 rr))]
// One thread per (l, rr) fiber: the K1 x K2 inputs are read once, the inner
// sums t(i1, k2) stay in registers, the r1 x r2 outputs are written once. Each
// sum runs in the same order with the same fma as k_small_ttm, so the result
// is bitwise that of the two separate passes (which read and write the
// intermediate through HBM).
constexpr int ST2_THREADS = 128, ST2_R1 = 8, ST2_T = 64;  // r1 <= 8, K2 * r1 <= 64
template <typename T>
__global__ void __launch_bounds__(ST2_THREADS) k_small_ttm2(const T* __restrict__ x, int64_t L, int K1, int K2,
                                                            int64_t Rr, const double* __restrict__ m1, int r1,
                                                            int64_t s1r, int64_t s1k, const double* __restrict__ m2,
                                                            int r2, int64_t s2r, int64_t s2k, double* __restrict__ y) {
  extern __shared__ double sm2[];
  double* A1 = sm2;                  // [k1][i1]
  double* A2 = A1 + K1 * r1;         // [k2][i2]
  double* tb = A2 + K2 * r2;         // per-thread t(i1, k2) at tb[(k2 * r1 + i1) * ST2_THREADS + tid]
  const int tid = threadIdx.x;
  for (int e = tid; e < K1 * r1; e += blockDim.x) A1[e] = m1[(e % r1) * s1r + (e / r1) * s1k];
  for (int e = tid; e < K2 * r2; e += blockDim.x) A2[e] = m2[(e % r2) * s2r + (e / r2) * s2k];
  __syncthreads();
  const int64_t total = L * Rr;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + tid; f < total; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = f % L, rr = f / L;
    const T* xp = x + l + L * (int64_t)K1 * K2 * rr;
    for (int k2 = 0; k2 < K2; ++k2) {  // first TTM: t(i1, k2) = sum_k1 M1(i1,k1) x(k1, k2)
      double acc[ST2_R1];
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i) acc[i] = 0.0;
      for (int k1 = 0; k1 < K1; ++k1) {
        const double xv = ld(xp, L * (k1 + (int64_t)K1 * k2));
#pragma unroll
        for (int i = 0; i < ST2_R1; ++i)
          if (i < r1) acc[i] = fma(A1[k1 * r1 + i], xv, acc[i]);
      }
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i)
        if (i < r1) tb[(k2 * r1 + i) * ST2_THREADS + tid] = acc[i];
    }
    double* yp = y + l + L * (int64_t)r1 * r2 * rr;
    for (int i2 = 0; i2 < r2; ++i2) {  // second TTM: y(i1, i2) = sum_k2 M2(i2,k2) t(i1, k2)
      double acc[ST2_R1];
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i) acc[i] = 0.0;
      for (int k2 = 0; k2 < K2; ++k2) {
        const double a = A2[k2 * r2 + i2];
#pragma unroll
        for (int i = 0; i < ST2_R1; ++i)
          if (i < r1) acc[i] = fma(a, tb[(k2 * r1 + i) * ST2_THREADS + tid], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i)
        if (i < r1) yp[L * (i + (int64_t)r1 * i2)] = acc[i];
    }
  }
}

// K9 fused epilogue: the last two (small) mode products of the reconstruction
// with the residual against the source tensor, sum (t - y)^2, instead of
// writing y. Same products, in the same order, as k_small_ttm2; the squared
// differences reduce per block (fixed order) into part[blockIdx.x].
template <typename TT>
__global__ void __launch_bounds__(ST2_THREADS) k_small_ttm2_resid(const double* __restrict__ x, int64_t L, int K1,
                                                                  int K2, int64_t Rr, const double* __restrict__ m1,
                                                                  int r1, int64_t s1r, int64_t s1k,
                                                                  const double* __restrict__ m2, int r2, int64_t s2r,
                                                                  int64_t s2k, const TT* __restrict__ t,
                                                                  double* __restrict__ part) {
  extern __shared__ double sm2[];
  __shared__ double red[ST2_THREADS / 32];
  double* A1 = sm2;
  double* A2 = A1 + K1 * r1;
  double* tb = A2 + K2 * r2;
  const int tid = threadIdx.x;
  for (int e = tid; e < K1 * r1; e += blockDim.x) A1[e] = m1[(e % r1) * s1r + (e / r1) * s1k];
  for (int e = tid; e < K2 * r2; e += blockDim.x) A2[e] = m2[(e % r2) * s2r + (e / r2) * s2k];
  __syncthreads();
  double ss = 0.0;
  const int64_t total = L * Rr;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + tid; f < total; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = f % L, rr = f / L;
    const double* xp = x + l + L * (int64_t)K1 * K2 * rr;
    for (int k2 = 0; k2 < K2; ++k2) {
      double acc[ST2_R1];
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i) acc[i] = 0.0;
      for (int k1 = 0; k1 < K1; ++k1) {
        const double xv = xp[L * (k1 + (int64_t)K1 * k2)];
#pragma unroll
        for (int i = 0; i < ST2_R1; ++i)
          if (i < r1) acc[i] = fma(A1[k1 * r1 + i], xv, acc[i]);
      }
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i)
        if (i < r1) tb[(k2 * r1 + i) * ST2_THREADS + tid] = acc[i];
    }
    const TT* tp = t + l + L * (int64_t)r1 * r2 * rr;
    for (int i2 = 0; i2 < r2; ++i2) {
      double acc[ST2_R1];
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i) acc[i] = 0.0;
      for (int k2 = 0; k2 < K2; ++k2) {
        const double a = A2[k2 * r2 + i2];
#pragma unroll
        for (int i = 0; i < ST2_R1; ++i)
          if (i < r1) acc[i] = fma(a, tb[(k2 * r1 + i) * ST2_THREADS + tid], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < ST2_R1; ++i)
        if (i < r1) {
          const double d = (double)tp[L * (i + (int64_t)r1 * i2)] - acc[i];
          ss = fma(d, d, ss);
        }
    }
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < ST2_THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// ---- small-mode Gram, pass 1: per-block partial upper-triangle sums.
constexpr int SG_THREADS = 256, SG_MAXPP = 9;  // K <= 64 -> 2080 pairs <= 9*256
template <typename T>
__global__ void __launch_bounds__(SG_THREADS) k_small_gram(const T* __restrict__ x, int64_t L, int K,
                                                           int64_t Rr, int TP, double* __restrict__ part) {
  extern __shared__ double sX[];  // [k][TP + 1]: odd row stride, so the K rows of one column sit in different banks
  __shared__ double red[SG_THREADS];
  const int npairs = K * (K + 1) / 2;
  const int G = npairs >= SG_THREADS ? 1 : SG_THREADS / npairs;
  const int tid = threadIdx.x;
  const int grp = npairs >= SG_THREADS ? 0 : tid / npairs;
  const int64_t P = L * Rr;
  const int TPS = TP + 1;
  double acc[SG_MAXPP];
#pragma unroll
  for (int q = 0; q < SG_MAXPP; ++q) acc[q] = 0.0;
  // pair index -> (i, j) with i <= j, row-major over the upper triangle
  for (int64_t p0 = (int64_t)blockIdx.x * TP; p0 < P; p0 += (int64_t)gridDim.x * TP) {
    __syncthreads();
    const int64_t l0 = p0 % L, rr0 = p0 / L;  // once per tile; elements step l, wrapping rarely
    for (int e = tid; e < TP * K; e += SG_THREADS) {
      const int k = e / TP, pp = e % TP;
      double v = 0.0;
      if (p0 + pp < P) {
        int64_t l = l0 + pp, rr = rr0;
        if (l >= L) { const int64_t w = l / L; l -= w * L; rr += w; }
        v = ld(x, l + L * (k + (int64_t)K * rr));
      }
      sX[k * TPS + pp] = v;
    }
    __syncthreads();
    if (npairs >= SG_THREADS) {
#pragma unroll
      for (int q = 0; q < SG_MAXPP; ++q) {
        const int pr = tid + q * SG_THREADS;
        if (pr < npairs) {
          int i = 0, rem = pr;
          while (rem >= K - i) { rem -= K - i; ++i; }
          const int j = i + rem;
          double s = 0.0;
          for (int pp = 0; pp < TP; ++pp) s = fma(sX[i * TPS + pp], sX[j * TPS + pp], s);
          acc[q] += s;
        }
      }
    } else if (tid < G * npairs) {
      const int pr = tid % npairs;
      int i = 0, rem = pr;
      while (rem >= K - i) { rem -= K - i; ++i; }
      const int j = i + rem;
      double s = 0.0;
      for (int pp = grp; pp < TP; pp += G) s = fma(sX[i * TPS + pp], sX[j * TPS + pp], s);
      acc[0] += s;
    }
  }
  // combine groups (fixed order) and write this block's partial
  if (npairs >= SG_THREADS) {
#pragma unroll
    for (int q = 0; q < SG_MAXPP; ++q) {
      const int pr = tid + q * SG_THREADS;
      if (pr < npairs) part[(int64_t)blockIdx.x * npairs + pr] = acc[q];
    }
  } else {
    red[tid] = acc[0];
    __syncthreads();
    if (tid < npairs) {
      double s = 0.0;
      for (int gq = 0; gq < G; ++gq) s += red[gq * npairs + tid];
      part[(int64_t)blockIdx.x * npairs + tid] = s;
    }
  }
}

// One warp per Gram pair: lanes take the block partials b = lane, lane+32, ...
// (independent loads), then a fixed shuffle tree -- deterministic.
__global__ void k_small_gram_reduce(const double* __restrict__ part, int nblk, int K, double* __restrict__ g) {
  const int npairs = K * (K + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int pr = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (pr >= npairs) return;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * npairs + pr];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    int i = 0, rem = pr;
    while (rem >= K - i) { rem -= K - i; ++i; }
    const int j = i + rem;
    g[i + (int64_t)K * j] = s;
    g[j + (int64_t)K * i] = s;
  }
}

// ---- reductions
template <typename T>
__global__ void k_sumsq_part(const T* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = ld(x, i);
    s = fma(v, v, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  // fixed assignment: thread t sums t, t+blockDim, ... then fixed tree
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_absmax_part(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fmax(s, fabs(x[i]));
  s = block_max(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_max_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s = fmax(s, part[i]);
  s = block_max(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_diff_part(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0, t = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    s = fma(d, d, s);
    t = fma(b[i], b[i], t);
  }
  s = block_sum(s, sh);
  t = block_sum(t, sh);
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = s; part[2 * blockIdx.x + 1] = t; }
}

__global__ void k_diff_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { s += part[2 * i]; t += part[2 * i + 1]; }
  s = block_sum(s, sh);
  t = block_sum(t, sh);
  if (threadIdx.x == 0) { out[0] = s; out[1] = t; }
}

template <typename T>
__global__ void k_resid_part(const T* __restrict__ t, const double* __restrict__ th, int64_t n,
                             double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = ld(t, i) - th[i];
    s = fma(d, d, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---- codec
__global__ void k_quant_step(const double* amax, double f, double* step) {
  // codec.py:124: amax * 2**((qp-51)/6) * 2**-8, evaluated left to right; f is
  // the host-libm value of 2**((qp-51)/6) so the step is bit-identical.
  const double a = *amax;
  *step = a > 0.0 ? (a * f) * 0x1p-8 : 1.0;
}

__global__ void k_quantize(const double* __restrict__ core, int64_t n, const double* __restrict__ step,
                           int64_t* __restrict__ lv) {
  const double s = *step;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double q = core[i] / s;                   // codec.py:126 core / step
    const double r = floor(fabs(q) + 0.5);          // codec.py:99 round half away
    lv[i] = (int64_t)(q > 0.0 ? r : (q < 0.0 ? -r : 0.0));
  }
}

__global__ void k_dequant(const int64_t* __restrict__ lv, int64_t n, double step, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)lv[i] * step;
}

// one warp per column: first index of max |v| made positive (tensor.py:203-209)
__global__ void k_sign_fix(double* __restrict__ v, int64_t n, int64_t k) {
  const int lane = threadIdx.x & 31;
  const int64_t col = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= k) return;
  double* c = v + col * n;
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t i = lane; i < n; i += 32) {
    const double a = fabs(c[i]);
    if (a > best) { best = a; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  const bool flip = c[bi] < 0.0;
  if (flip)
    for (int64_t i = lane; i < n; i += 32) c[i] = -c[i];
}

__global__ void k_copy(double* __restrict__ d, const double* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void k_f32_f64(const float* __restrict__ s, double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = (double)s[i];
}

__global__ void k_id_combo(const double* __restrict__ w, int64_t n, double a, double b, double* __restrict__ o) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    o[e] = b * w[e] + (i == j ? a : 0.0);
  }
}

__global__ void k_offid_part(const double* __restrict__ w, int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    s = fmax(s, fabs(w[e] - (i == j ? 1.0 : 0.0)));
  }
  s = block_max(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

inline int grid_for(Ctx& c, int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 16LL * c.num_sms));
}

#define LAUNCHED(name) do { c.launches++; check_launch(name); } while (0)

}  // namespace

void small_ttm(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t Rr, const double* m, int64_t r,
               int64_t sMr, int64_t sMk, double* y) {
  const int64_t nch = ceil_div(r, 8);
  const int64_t total = L * Rr * nch;
  if (total == 0) return;
  const size_t smem = sizeof(double) * K * r;
  const int blocks = grid_for(c, total);
  if (tx == F32)
    k_small_ttm<float><<<blocks, 256, smem, c.stream>>>((const float*)x, L, (int)K, Rr, m, (int)r, sMr, sMk, y);
  else
    k_small_ttm<double><<<blocks, 256, smem, c.stream>>>((const double*)x, L, (int)K, Rr, m, (int)r, sMr, sMk, y);
  LAUNCHED("k_small_ttm");
}

bool small_ttm2(Ctx& c, const void* x, DType tx, int64_t L, int64_t K1, int64_t K2, int64_t Rr, const double* m1,
                int64_t r1, int64_t s1r, int64_t s1k, const double* m2, int64_t r2, int64_t s2r, int64_t s2k,
                double* y) {
  if (r1 > ST2_R1 || K2 * r1 > ST2_T || K1 > 64 || K2 > 64 || r2 > 64) return false;
  const int64_t total = L * Rr;
  if (total == 0) return true;
  const size_t smem = sizeof(double) * (K1 * r1 + K2 * r2 + (size_t)K2 * r1 * ST2_THREADS);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, ST2_THREADS), 32LL * c.num_sms));
  // > 48 KB of per-thread inner sums (e.g. view-exposure 18 -> 9)
  set_smem_attr(c, tx == F32 ? (const void*)k_small_ttm2<float> : (const void*)k_small_ttm2<double>,
                sizeof(double) * (64 * 8 + 64 * 64 + (size_t)ST2_T * ST2_THREADS));
  if (tx == F32)
    k_small_ttm2<float><<<blocks, ST2_THREADS, smem, c.stream>>>((const float*)x, L, (int)K1, (int)K2, Rr, m1,
                                                                  (int)r1, s1r, s1k, m2, (int)r2, s2r, s2k, y);
  else
    k_small_ttm2<double><<<blocks, ST2_THREADS, smem, c.stream>>>((const double*)x, L, (int)K1, (int)K2, Rr, m1,
                                                                   (int)r1, s1r, s1k, m2, (int)r2, s2r, s2k, y);
  LAUNCHED("k_small_ttm2");
  return true;
}

bool small_ttm2_resid(Ctx& c, const double* x, int64_t L, int64_t K1, int64_t K2, int64_t Rr, const double* m1,
                      int64_t r1, int64_t s1r, int64_t s1k, const double* m2, int64_t r2, int64_t s2r, int64_t s2k,
                      const void* t, DType tt, double* out_dev) {
  if (r1 > ST2_R1 || K2 * r1 > ST2_T || K1 > 64 || K2 > 64 || r2 > 64) return false;
  const int64_t total = L * Rr;
  const size_t smem = sizeof(double) * (K1 * r1 + K2 * r2 + (size_t)K2 * r1 * ST2_THREADS);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, ST2_THREADS), 8LL * c.num_sms));
  const void* fn = tt == F32 ? (const void*)k_small_ttm2_resid<float> : (const void*)k_small_ttm2_resid<double>;
  set_smem_attr(c, fn, sizeof(double) * (64 * 8 + 64 * 64 + (size_t)ST2_T * ST2_THREADS));
  double* part = alloc<double>(c, (size_t)blocks);
  if (tt == F32)
    k_small_ttm2_resid<float><<<blocks, ST2_THREADS, smem, c.stream>>>(x, L, (int)K1, (int)K2, Rr, m1, (int)r1, s1r,
                                                                        s1k, m2, (int)r2, s2r, s2k,
                                                                        (const float*)t, part);
  else
    k_small_ttm2_resid<double><<<blocks, ST2_THREADS, smem, c.stream>>>(x, L, (int)K1, (int)K2, Rr, m1, (int)r1,
                                                                         s1r, s1k, m2, (int)r2, s2r, s2k,
                                                                         (const double*)t, part);
  LAUNCHED("k_small_ttm2_resid");
  k_sum_final<<<1, 1024, 0, c.stream>>>(part, blocks, out_dev);
  LAUNCHED("k_sum_final");
  return true;
}

void small_gram(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t Rr, double* g) {
  const int npairs = (int)(K * (K + 1) / 2);
  int TP = (int)std::max<int64_t>(32, std::min<int64_t>(1024, 4096 / K));  // <= 32 KB dynamic smem
  TP = (TP / 32) * 32;
  const int64_t P = L * Rr;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(P, TP), 2LL * c.num_sms));
  double* part = alloc<double>(c, (size_t)nblk * npairs);
  const size_t smem = sizeof(double) * (TP + 1) * K;
  if (tx == F32)
    k_small_gram<float><<<nblk, SG_THREADS, smem, c.stream>>>((const float*)x, L, (int)K, Rr, TP, part);
  else
    k_small_gram<double><<<nblk, SG_THREADS, smem, c.stream>>>((const double*)x, L, (int)K, Rr, TP, part);
  LAUNCHED("k_small_gram");
  k_small_gram_reduce<<<(unsigned)ceil_div((int64_t)npairs * 32, 256), 256, 0, c.stream>>>(part, nblk, (int)K, g);
  LAUNCHED("k_small_gram_reduce");
}

void sumsq_async(Ctx& c, const void* x, DType tx, int64_t n, double* out_dev) {
  double* part = alloc<double>(c, RED_BLOCKS);
  if (tx == F32) k_sumsq_part<float><<<RED_BLOCKS, 256, 0, c.stream>>>((const float*)x, n, part);
  else k_sumsq_part<double><<<RED_BLOCKS, 256, 0, c.stream>>>((const double*)x, n, part);
  LAUNCHED("k_sumsq_part");
  k_sum_final<<<1, 1024, 0, c.stream>>>(part, RED_BLOCKS, out_dev);
  LAUNCHED("k_sum_final");
}

double sumsq(Ctx& c, const void* x, DType tx, int64_t n) {
  const size_t m = c.arena.mark();
  double* d = alloc<double>(c, 1);
  sumsq_async(c, x, tx, n, d);
  TMB_CUDA(cudaMemcpyAsync(c.host_pinned, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  c.arena.release(m);
  return c.host_pinned[0];
}

void resid2_async(Ctx& c, const void* t, DType tt, const double* th, int64_t n, double* out_dev) {
  double* part = alloc<double>(c, RED_BLOCKS);
  if (tt == F32) k_resid_part<float><<<RED_BLOCKS, 256, 0, c.stream>>>((const float*)t, th, n, part);
  else k_resid_part<double><<<RED_BLOCKS, 256, 0, c.stream>>>((const double*)t, th, n, part);
  LAUNCHED("k_resid_part");
  k_sum_final<<<1, 1024, 0, c.stream>>>(part, RED_BLOCKS, out_dev);
  LAUNCHED("k_sum_final");
}

void absmax_async(Ctx& c, const double* x, int64_t n, double* out_dev) {
  double* part = alloc<double>(c, RED_BLOCKS);
  k_absmax_part<<<RED_BLOCKS, 256, 0, c.stream>>>(x, n, part);
  LAUNCHED("k_absmax_part");
  k_max_final<<<1, 1024, 0, c.stream>>>(part, RED_BLOCKS, out_dev);
  LAUNCHED("k_max_final");
}

void quant_step(Ctx& c, const double* amax_dev, int qp, double* step_dev) {
  const double f = std::pow(2.0, (qp - 51) / 6.0);
  k_quant_step<<<1, 1, 0, c.stream>>>(amax_dev, f, step_dev);
  LAUNCHED("k_quant_step");
}

void quantize(Ctx& c, const double* core, int64_t n, const double* step_dev, int64_t* levels) {
  if (n == 0) return;
  k_quantize<<<grid_for(c, n), 256, 0, c.stream>>>(core, n, step_dev, levels);
  LAUNCHED("k_quantize");
}

void dequant(Ctx& c, const int64_t* lv, int64_t n, double step, double* out) {
  if (n == 0) return;
  k_dequant<<<grid_for(c, n), 256, 0, c.stream>>>(lv, n, step, out);
  LAUNCHED("k_dequant");
}

void sign_fix(Ctx& c, double* v, int64_t n, int64_t k) {
  if (k == 0 || n == 0) return;
  k_sign_fix<<<(unsigned)ceil_div(k, 8), 256, 0, c.stream>>>(v, n, k);
  LAUNCHED("k_sign_fix");
}

void diff_norms(Ctx& c, const double* a, const double* b, int64_t n, double* out2_dev) {
  constexpr int NB = 256;
  double* part = alloc<double>(c, 2 * NB);
  k_diff_part<<<NB, 256, 0, c.stream>>>(a, b, n, part);
  LAUNCHED("k_diff_part");
  k_diff_final<<<1, 256, 0, c.stream>>>(part, NB, out2_dev);
  LAUNCHED("k_diff_final");
}

void copy_d(Ctx& c, double* dst, const double* src, int64_t n) {
  if (n == 0) return;
  k_copy<<<grid_for(c, n), 256, 0, c.stream>>>(dst, src, n);
  LAUNCHED("k_copy");
}

void axpy(Ctx& c, int64_t n, double alpha, const double* x, double* y) {
  if (n == 0) return;
  k_axpy<<<grid_for(c, n), 256, 0, c.stream>>>(n, alpha, x, y);
  LAUNCHED("k_axpy");
}

void convert_f32_f64(Ctx& c, const float* s, double* d, int64_t n) {
  if (n == 0) return;
  k_f32_f64<<<grid_for(c, n), 256, 0, c.stream>>>(s, d, n);
  LAUNCHED("k_f32_f64");
}

void scale_identity_combo(Ctx& c, const double* w, int64_t n, double a, double b, double* out) {
  k_id_combo<<<grid_for(c, n * n), 256, 0, c.stream>>>(w, n, a, b, out);
  LAUNCHED("k_id_combo");
}

void maxabs_offidentity(Ctx& c, const double* w, int64_t n, double* out_dev) {
  constexpr int NB = 128;
  double* part = alloc<double>(c, NB);
  k_offid_part<<<NB, 256, 0, c.stream>>>(w, n, part);
  LAUNCHED("k_offid_part");
  k_max_final<<<1, 128, 0, c.stream>>>(part, NB, out_dev);
  LAUNCHED("k_max_final");
}

}  // namespace tmb
