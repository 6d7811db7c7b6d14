// Ozaki-split fp64-equivalent TTM on the 5th-gen tensor cores (tcgen05.mma kind::i8).
//
// y = x x_n M  (ttm, tensor.py:111-123) for the full passes over the tensor.
// GEMM view: rows m = (i, l) of x (i < L = prod(dims before n), l < R = prod
// dims after n), K = dims[n], N = rows of M:  C(m, r) = sum_k A(m, k) B(k, r)
// with A(m, k) = x[i + L k + L K l], B(k, r) = M(r, k).
//
// Split (Ozaki scheme, int8 digits): each row of A and each column of B is
// scaled by a power of two 2^e so its entries lie in (-1, 1), then written as
// 8 signed digits a = d0 2^-6 + sum_{s>=1} d_s 2^(-6-7s), |d| <= 64 (55 bits,
// >= the 53 of an fp64 mantissa). A(m,k) B(k,r) then is a sum of digit
// products d_s f_t 2^(-12-7(s+t)); the 36 products with s + t < 8 are kept
// (the first dropped group is 2^-56 below the leading one, the fp64 GEMM's own
// rounding level), each shift group g = s + t accumulating exactly in int32
// (|d f| <= 2^12, <= 8 pairs per group, K <= 2^16).
//
// Kernel: one CTA per 128 (factor rows) x 64 (tensor rows) output tile,
// warp-specialised. Lane 0 of warp 0 streams 64-byte K chunks of all 8 factor
// digit planes (128 rows) and all 8 tensor digit planes (64 rows) with one 3-D TMA each (SWIZZLE_64B, the canonical
// K-major SW64 UMMA layout) into a 2-stage ring; lane 0 of warp 1 issues the 72
// tcgen05.mma (M=128, N=64, K=32) per chunk into 8 TMEM accumulators (8 x 64
// of the 512 columns), one per shift group, committing each stage back to the
// producer; then all 4 warps read the accumulators (tcgen05.ld 32x32b), form
// sum_g acc_g 2^(-12-7g) in fp64, apply 2^(e_r + e_m) and store y. The grid
// runs the factor-row tiles fastest, so the CTAs sharing a tensor tile read its
// digit planes from HBM once (the factor digits stay in L2).
#include <cuda.h>

#include <cstdlib>

#include "tmb_internal.cuh"

namespace tmb {
namespace {

constexpr int OZ_S = 8;                                   // digits per operand
constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 64, OZ_ST = 2, OZ_NT = 128;
constexpr uint32_t OZ_A_BYTES = OZ_S * OZ_BM * OZ_BK;    // 64 KB
constexpr uint32_t OZ_B_BYTES = OZ_S * OZ_BN * OZ_BK;    // 32 KB
constexpr uint32_t OZ_STAGE = OZ_A_BYTES + OZ_B_BYTES;  // 96 KB

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// v 2^(55-e) rounded to an integer (|v| < 2^e): one rounding at 2^-55 of the
// row/column maximum. fp32 inputs take an integer-only path from the bit pattern.
__device__ __forceinline__ long long fixed55(double v, int e) { return __double2ll_rn(ldexp(v, 55 - e)); }
__device__ __forceinline__ long long fixed55(float v, int e) {
  const uint32_t b = __float_as_uint(v);
  const int ex = (int)((b >> 23) & 0xFF);
  long long mant = (long long)(b & 0x7FFFFF);
  int sh;
  if (ex == 0) sh = 1 - 150 + 55 - e;  // subnormal
  else { mant |= 0x800000; sh = ex - 150 + 55 - e; }
  long long a;
  if (sh >= 0) a = mant << sh;
  else if (sh > -40) a = (mant + (1LL << (-sh - 1))) >> (-sh);  // round half up (ties are measure-zero)
  else a = 0;
  return (b >> 31) ? -a : a;
}

// balanced 7-bit digits of the fixed-point value: a = sum_s d_s 2^(-6-7s), |d_s| <= 64
template <typename T>
__device__ __forceinline__ void digits8(T v, int e, int8_t (&d)[OZ_S]) {
  long long A = fixed55(v, e);
#pragma unroll
  for (int s = 0; s < OZ_S - 1; ++s) {
    const int sh = 49 - 7 * s;
    const long long q = (A + (1LL << (sh - 1))) >> sh;
    d[s] = (int8_t)q;
    A -= q << sh;
  }
  d[OZ_S - 1] = (int8_t)A;
}

__device__ __forceinline__ int exp_of(double mx) {  // smallest e with mx < 2^e (0 for mx == 0)
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);
  return e;
}

template <typename T>
__device__ __forceinline__ double ldv(const T* p, int64_t i) { return (double)p[i]; }
template <typename T>
__device__ __forceinline__ T ldraw(const T* p, int64_t i) { return p[i]; }

// row exponents of the x operand, rows m = (i, l): for L >= 32 a block covers 32
// consecutive rows (lanes, coalesced along i) and its 8 warps split K; else a
// warp per row with lanes along k
template <typename T>
__global__ void __launch_bounds__(256) k_oz_rowexp(const T* __restrict__ x, int64_t L, int64_t K, int64_t R,
                                                   int* __restrict__ ea) {
  const int64_t M = L * R;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (L >= 32) {
    __shared__ double red[8][32];
    const int64_t m = (int64_t)blockIdx.x * 32 + lane;
    double mx = 0.0;
    if (m < M) {
      const int64_t i = m % L, l = m / L;
      const T* p = x + i + L * K * l;
      // 8 independent loads in flight per thread (the pass is latency-bound otherwise)
      double mq[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int64_t k = w;
      for (; k + 56 < K; k += 64) {
#pragma unroll
        for (int q = 0; q < 8; ++q) mq[q] = fmax(mq[q], fabs(ldv(p, L * (k + 8 * q))));
      }
      for (; k < K; k += 8) mq[0] = fmax(mq[0], fabs(ldv(p, L * k)));
#pragma unroll
      for (int q = 0; q < 8; ++q) mx = fmax(mx, mq[q]);
    }
    red[w][lane] = mx;
    __syncthreads();
    if (w == 0 && m < M) {
      for (int q = 1; q < 8; ++q) mx = fmax(mx, red[q][lane]);
      ea[m] = exp_of(mx);
    }
  } else {
    const int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (m >= M) return;
    const int64_t i = m % L, l = m / L;
    const T* p = x + i + L * K * l;
    double mq[4] = {0, 0, 0, 0};
    int64_t k = lane;
    for (; k + 96 < K; k += 128) {
#pragma unroll
      for (int q = 0; q < 4; ++q) mq[q] = fmax(mq[q], fabs(ldv(p, L * (k + 32 * q))));
    }
    for (; k < K; k += 32) mq[0] = fmax(mq[0], fabs(ldv(p, L * k)));
    double mx = fmax(fmax(mq[0], mq[1]), fmax(mq[2], mq[3]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) ea[m] = exp_of(mx);
  }
}

// fp32 rows with L % 4 == 0: each lane covers 4 consecutive rows (i..i+3 of one
// slab l) with 16-byte loads, so a block covers 128 rows; 8 warps split K.
__global__ void __launch_bounds__(256) k_oz_rowexp_v4(const float* __restrict__ x, int64_t L, int64_t K, int64_t R,
                                                      int* __restrict__ ea) {
  __shared__ float red[8][128];
  const int64_t M = L * R;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t m = (int64_t)blockIdx.x * 128 + 4 * lane;  // first of this lane's 4 rows
  float4 mx = make_float4(0.f, 0.f, 0.f, 0.f);
  if (m < M) {
    const int64_t i = m % L, l = m / L;
    const float* p = x + i + L * K * l;
    float4 mq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) mq[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t k = w;
    for (; k + 24 < K; k += 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p + L * (k + 8 * q)));
        mq[q].x = fmaxf(mq[q].x, fabsf(v.x)); mq[q].y = fmaxf(mq[q].y, fabsf(v.y));
        mq[q].z = fmaxf(mq[q].z, fabsf(v.z)); mq[q].w = fmaxf(mq[q].w, fabsf(v.w));
      }
    }
    for (; k < K; k += 8) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + L * k));
      mq[0].x = fmaxf(mq[0].x, fabsf(v.x)); mq[0].y = fmaxf(mq[0].y, fabsf(v.y));
      mq[0].z = fmaxf(mq[0].z, fabsf(v.z)); mq[0].w = fmaxf(mq[0].w, fabsf(v.w));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mx.x = fmaxf(mx.x, mq[q].x); mx.y = fmaxf(mx.y, mq[q].y);
      mx.z = fmaxf(mx.z, mq[q].z); mx.w = fmaxf(mx.w, mq[q].w);
    }
  }
  red[w][4 * lane] = mx.x; red[w][4 * lane + 1] = mx.y; red[w][4 * lane + 2] = mx.z; red[w][4 * lane + 3] = mx.w;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int64_t mm = (int64_t)blockIdx.x * 128 + threadIdx.x;
    float v = red[0][threadIdx.x];
    for (int q = 1; q < 8; ++q) v = fmaxf(v, red[q][threadIdx.x]);
    if (mm < M) ea[mm] = exp_of((double)v);  // max of exact fp32 magnitudes: same exponent as the fp64 path
  }
}

// x digits, K-major planes SA[s][m][k] (Mp x Kp, zero padded). Tiles of 32 rows
// x 128 k through shared memory: reads coalesce along the contiguous index (i
// when L >= 32, else k), writes are 4 packed digits (32 bits) per lane, 128 B per
// plane row.
template <typename T>
__global__ void __launch_bounds__(256) k_oz_sliceA(const T* __restrict__ x, int64_t L, int64_t K, int64_t R,
                                                   const int* __restrict__ ea, int64_t Mp, int64_t Kp,
                                                   int8_t* __restrict__ sa) {
  __shared__ __align__(16) int8_t tile[OZ_S][32][128 + 4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 8 warps
  const int64_t M = L * R;
  const int64_t m0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 128;
  if (L >= 32) {  // lanes along m (i contiguous), warps over k
    const int64_t m = m0 + lane;
    const bool mok = m < M;
    const int64_t i = mok ? m % L : 0, l = mok ? m / L : 0;
    const int e = mok ? ea[m] : 0;
    T xv[16];  // all 16 loads of this thread in flight before any digit work
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t k = k0 + w + 8 * q;
      xv[q] = (mok && k < K) ? ldraw(x, i + L * k + L * K * l) : (T)0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int kk = w + 8 * q;
      int8_t d[OZ_S];
      digits8(xv[q], e, d);
#pragma unroll
      for (int s2 = 0; s2 < OZ_S; ++s2) tile[s2][lane][kk] = d[s2];
    }
  } else {  // lanes along k, warps over m
    T xv[4][4];
    int ev[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {  // all 16 loads first
      const int64_t m = m0 + w + 8 * a;
      const bool mok = m < M;
      const int64_t i = mok ? m % L : 0, l = mok ? m / L : 0;
      ev[a] = mok ? ea[m] : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t k = k0 + lane + 32 * q;
        xv[a][q] = (mok && k < K) ? ldraw(x, i + L * k + L * K * l) : (T)0;
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int8_t d[OZ_S];
        digits8(xv[a][q], ev[a], d);
#pragma unroll
        for (int s2 = 0; s2 < OZ_S; ++s2) tile[s2][w + 8 * a][lane + 32 * q] = d[s2];
      }
  }
  __syncthreads();
  for (int mm = w; mm < 32; mm += 8) {
    const int64_t m = m0 + mm, k = k0 + 4 * lane;
    if (m >= Mp || k >= Kp) continue;
#pragma unroll
    for (int s2 = 0; s2 < OZ_S; ++s2) {
      const uint32_t v = (uint32_t)(uint8_t)tile[s2][mm][4 * lane] | ((uint32_t)(uint8_t)tile[s2][mm][4 * lane + 1] << 8) |
                         ((uint32_t)(uint8_t)tile[s2][mm][4 * lane + 2] << 16) |
                         ((uint32_t)(uint8_t)tile[s2][mm][4 * lane + 3] << 24);
      *reinterpret_cast<uint32_t*>(sa + ((int64_t)s2 * Mp + m) * Kp + k) = v;
    }
  }
}

// B(k, n) = mat[n sMr + k sMk]: column exponents (warp per column) and digits SB[t][n][k]
__global__ void k_oz_colexp(const double* __restrict__ mat, int64_t K, int64_t N, int64_t sMr, int64_t sMk,
                            int* __restrict__ eb) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (n >= N) return;
  double mx = 0.0;
  for (int64_t k = lane; k < K; k += 32) mx = fmax(mx, fabs(mat[n * sMr + k * sMk]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) eb[n] = exp_of(mx);
}

__global__ void k_oz_sliceB(const double* __restrict__ mat, int64_t K, int64_t N, int64_t sMr, int64_t sMk,
                            const int* __restrict__ eb, int64_t Np, int64_t Kp, int8_t* __restrict__ sb) {
  const int64_t total = Np * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e % Kp, n = e / Kp;
    int8_t d[OZ_S] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (n < N && k < K) digits8(mat[n * sMr + k * sMk], eb[n], d);
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) sb[((int64_t)s * Np + n) * Kp + k] = d[s];
  }
}

__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;        // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                 // descriptor version (sm100)
  d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;        // SBO: 8 rows x 32 B
  d |= (uint64_t)1 << 46;                 // descriptor version (sm100)
  d |= (uint64_t)6 << 61;                 // SWIZZLE_32B
  return d;
}

// One elected lane of a CONVERGED warp. The tcgen05 / TMA issue code runs under this
// predicate instead of `lane == 0`: in a plain divergent branch ptxas wraps every uniform-
// datapath instruction (UTCIMMA, UTMALDG) in an ELECT / BRA.U.ANY loop over the active
// lanes -- ~7 dependent instructions and a branch per MMA, 69 cycles per MMA issued against
// the 34 the tensor pipe needs (ncu source view: the issuing thread 70 % in that loop).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (long long it = 0; it < 2000000000LL; ++it) {
    uint32_t done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
  }
  asm volatile("trap;");  // a protocol bug must not hang the GPU
}

// Epilogue shared by both GEMM variants: warp w holds factor rows r = m0 + 32w
// + lane (TMEM lanes); columns are tensor rows m = (i, l), 8 at a time. Forms
// sum_g acc_g 2^(-12-7g) in fp64 (exact-constant FMAs, small groups first),
// scales by 2^(e_r + e_m) (built from the exponent bits when normal) and
// stores 8 consecutive i of y for one r; (i, l) advance incrementally (one
// division per CTA, then wrap-around steps).
template <int BN>
__device__ __forceinline__ void oz_epilogue(uint32_t tmem, int warp, int lane, int64_t m0, int64_t n0,
                                            const int* __restrict__ eu, const int* __restrict__ ex, int64_t L,
                                            int64_t R, int64_t N, double* __restrict__ y) {
  const int64_t r = m0 + warp * 32 + lane;
  const bool rok = r < N;
  const int er = rok ? eu[r] : 0;
  const int64_t MX = L * R;
  int64_t ib = n0 % L, lb = n0 / L;  // (i, l) of column c0
  for (int c0 = 0; c0 < BN; c0 += 8) {
    uint32_t v[OZ_S][8];
#pragma unroll
    for (int g = 0; g < OZ_S; ++g)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[g][0]), "=r"(v[g][1]), "=r"(v[g][2]), "=r"(v[g][3]), "=r"(v[g][4]), "=r"(v[g][5]),
                     "=r"(v[g][6]), "=r"(v[g][7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(g * BN + c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (rok) {
      int64_t i = ib, l = lb;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t m = n0 + c0 + j;
        if (m < MX) {
          double acc = 0.0;
#pragma unroll
          for (int g = OZ_S - 1; g >= 0; --g)
            acc = fma((double)(int32_t)v[g][j], __longlong_as_double((long long)(1023 - 12 - 7 * g) << 52), acc);
          const int E = er + __ldg(ex + m);
          const double out = (E >= -1022 && E <= 1023) ? acc * __longlong_as_double((long long)(E + 1023) << 52)
                                                        : ldexp(acc, E);
          y[i + L * r + L * N * l] = out;
        }
        if (++i == L) { i = 0; ++l; }
      }
    }
    ib += 8;
    while (ib >= L) { ib -= L; ++lb; }
  }
}

// A operand (UMMA M side, 128 rows): factor digit planes, rows r (exponents eu);
// B operand (UMMA N side, 64 rows): tensor digit planes, rows m = (i, l) (exponents ex).
// The tensor digits -- the large operand -- are re-read once per 128 factor rows.
// BKB: bytes of K per pipeline stage -- 64 (SWIZZLE_64B, 2 stages of 96 KB, two
// K=32 MMAs per digit pair) or 32 (SWIZZLE_32B, 4 stages of 48 KB, one MMA).
template <int BKB>
__global__ void __launch_bounds__(OZ_NT, 1) k_oz_gemm(const __grid_constant__ CUtensorMap ta,
                                                      const __grid_constant__ CUtensorMap tb,
                                                      const int* __restrict__ eu, const int* __restrict__ ex,
                                                      int64_t L, int64_t R, int64_t N, int64_t Kp,
                                                      double* __restrict__ y) {
  constexpr int OZ_ST = BKB == 64 ? 2 : 4, OZ_BK = BKB, NH = BKB / 32;
  constexpr uint32_t OZ_A_BYTES = OZ_S * OZ_BM * BKB, OZ_STAGE = OZ_S * (OZ_BM + OZ_BN) * BKB;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[OZ_ST], empty[OZ_ST], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // factor-row tiles fastest: the CTAs sharing one tensor tile run together, so
  // its digit planes are read from HBM once and from L2 by the others
  const int64_t m0 = (int64_t)blockIdx.x * OZ_BM, n0 = (int64_t)blockIdx.y * OZ_BN;
  const int KT = (int)(Kp / OZ_BK);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < OZ_ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && elect_one()) {  // TMA producer: all 8 digit planes of A and of B per K chunk
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % OZ_ST;
      if (kt >= OZ_ST) mbar_wait(saddr(&empty[st]), ((kt / OZ_ST) - 1) & 1);
      const uint32_t fb = saddr(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(OZ_STAGE) : "memory");
      const uint32_t da = saddr(sm + st * OZ_STAGE), db = da + OZ_A_BYTES;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(da), "l"(&ta), "r"(kt * OZ_BK), "r"((int)m0), "r"(0), "r"(fb) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(db), "l"(&tb), "r"(kt * OZ_BK), "r"((int)n0), "r"(0), "r"(fb) : "memory");
    }
  } else if (warp == 1 && elect_one()) {  // MMA issuer: 36 digit pairs x 2 K-halves per chunk
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                           ((uint32_t)(OZ_BM >> 4) << 24);
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % OZ_ST;
      mbar_wait(saddr(&full[st]), (kt / OZ_ST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = saddr(sm + st * OZ_STAGE), b0 = a0 + OZ_A_BYTES;
      // descriptors differ only in the 14-bit start-address field (16-byte units):
      // build each stage's base once, add compile-time plane / K-half offsets
      const uint64_t adb = BKB == 64 ? sdesc_sw64(a0) : sdesc_sw32(a0);
      const uint64_t bdb = BKB == 64 ? sdesc_sw64(b0) : sdesc_sw32(b0);
#pragma unroll
      for (int g = 0; g < OZ_S; ++g) {
#pragma unroll
        for (int s = 0; s <= g; ++s) {
          const int t = g - s;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const uint64_t ad = adb + (uint64_t)((s * (OZ_BM * OZ_BK) + h * 32) >> 4);
            const uint64_t bd = bdb + (uint64_t)((t * (OZ_BN * OZ_BK) + h * 32) >> 4);
            const uint32_t acc = (kt > 0 || s > 0 || h > 0) ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                ::"r"(tmem + (uint32_t)(g * OZ_BN)), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(saddr(&empty[st])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&done)));
  }
  __syncwarp();
  mbar_wait(saddr(&done), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w holds factor rows r = m0 + 32w + lane (TMEM lanes); columns are
  // tensor rows (i, l), 8 at a time -> 8 consecutive i of y for one r
  oz_epilogue<OZ_BN>(tmem, warp, lane, m0, n0, eu, ex, L, R, N, y);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- N = 128 variant
// Same products, tiles of 128 factor rows x 128 tensor rows. Eight 128-column
// shift-group accumulators would need 1024 TMEM columns, so the 36 digit
// products run in three K passes over two halves of TMEM:
//   hi-1: s in 0..3, t = g - s for g in 4..7 (16 products; A planes 0-3, B planes 1-7)
//   hi-2: s in 4..7, t = g - s for g in 4..7 (10 products; A planes 4-7, B planes 0-3)
//   lo:   g in 0..3, s + t = g              (10 products; A planes 0-3, B planes 0-3)
// Groups 4-7 (hi) accumulate in TMEM columns (g-4)*128; after hi-2 the four
// epilogue warps fold them into sum_{g=7..4} acc_g 2^(-12-7g) and park that
// partial in y, TMEM is handed back, lo reuses it for groups 0-3, and the
// final epilogue continues the same fma chain (g = 3..0) from the parked
// partial before the 2^(e_r+e_m) scaling -- bitwise the N = 64 kernel's sum.
// Per 128x128x32 MMA the tensor core reads 8 KB of shared memory (4 KB per
// operand) against 6 KB per 128x64x32 before: the operand port was the bound.
// Warps: 0-3 epilogue (TMEM lane quarters), 4 TMA producer, 5 MMA issuer.
constexpr int OZ2_BN = 128, OZ2_NT = 192, OZ2_ST = 2;
constexpr uint32_t OZ2_PLANE = 128 * OZ_BK;              // 8 KB: one digit plane of a 128-row tile
constexpr uint32_t OZ2_STAGE = 4 * OZ2_PLANE + 7 * OZ2_PLANE;  // 88 KB (A 4 planes + B up to 7)

template <int PHASE>  // 0: groups 7..4 -> partial into y; 1: partial + groups 3..0, scaled
__device__ __forceinline__ void oz2_epilogue(uint32_t tmem, int warp, int lane, int64_t m0, int64_t n0,
                                             const int* __restrict__ eu, const int* __restrict__ ex, int64_t L,
                                             int64_t R, int64_t N, double* __restrict__ y) {
  const int64_t r = m0 + warp * 32 + lane;
  const bool rok = r < N;
  const int er = rok ? eu[r] : 0;
  const int64_t MX = L * R;
  int64_t ib = n0 % L, lb = n0 / L;
  for (int c0 = 0; c0 < OZ2_BN; c0 += 8) {
    uint32_t v[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[q][0]), "=r"(v[q][1]), "=r"(v[q][2]), "=r"(v[q][3]), "=r"(v[q][4]), "=r"(v[q][5]),
                     "=r"(v[q][6]), "=r"(v[q][7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(q * OZ2_BN + c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (rok) {
      int64_t i = ib, l = lb;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t m = n0 + c0 + j;
        if (m < MX) {
          double* yp = y + i + L * r + L * N * l;
          double acc = PHASE == 0 ? 0.0 : *yp;
#pragma unroll
          for (int q = 3; q >= 0; --q) {  // TMEM slot q holds group q + 4 (PHASE 0) or q (PHASE 1)
            const int g = PHASE == 0 ? q + 4 : q;
            acc = fma((double)(int32_t)v[q][j], __longlong_as_double((long long)(1023 - 12 - 7 * g) << 52), acc);
          }
          if (PHASE == 0) {
            *yp = acc;
          } else {
            const int E = er + __ldg(ex + m);
            *yp = (E >= -1022 && E <= 1023) ? acc * __longlong_as_double((long long)(E + 1023) << 52)
                                            : ldexp(acc, E);
          }
        }
        if (++i == L) { i = 0; ++l; }
      }
    }
    ib += 8;
    while (ib >= L) { ib -= L; ++lb; }
  }
}

__global__ void __launch_bounds__(OZ2_NT, 1) k_oz_gemm2(const __grid_constant__ CUtensorMap ta4,
                                                        const __grid_constant__ CUtensorMap tb7,
                                                        const __grid_constant__ CUtensorMap tb4,
                                                        const int* __restrict__ eu, const int* __restrict__ ex,
                                                        int64_t L, int64_t R, int64_t N, int64_t Kp,
                                                        double* __restrict__ y) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[OZ2_ST], empty[OZ2_ST], done_hi, done_lo, tmem_free;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * OZ_BM, n0 = (int64_t)blockIdx.y * OZ2_BN;
  const int KT = (int)(Kp / OZ_BK);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int st = 0; st < OZ2_ST; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[st])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[st])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&done_hi)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&done_lo)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(saddr(&tmem_free)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const int NQ = 3 * KT;  // chunk sequence: hi-1 (KT), hi-2 (KT), lo (KT)

  if (warp == 4) {
    if (elect_one()) {  // TMA producer
      for (int q = 0; q < NQ; ++q) {
        const int ph = q / KT, kt = q % KT, st = q % OZ2_ST;
        if (q >= OZ2_ST) mbar_wait(saddr(&empty[st]), ((q / OZ2_ST) - 1) & 1);
        const uint32_t fb = saddr(&full[st]);
        const uint32_t bytes = ph == 0 ? OZ2_STAGE : 8 * OZ2_PLANE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bytes) : "memory");
        const uint32_t da = saddr(sm + st * OZ2_STAGE), db = da + 4 * OZ2_PLANE;
        const int pa = ph == 1 ? 4 : 0;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(da), "l"(&ta4), "r"(kt * OZ_BK), "r"((int)m0), "r"(pa), "r"(fb) : "memory");
        if (ph == 0)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
              ::"r"(db), "l"(&tb7), "r"(kt * OZ_BK), "r"((int)n0), "r"(1), "r"(fb) : "memory");
        else
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
              ::"r"(db), "l"(&tb4), "r"(kt * OZ_BK), "r"((int)n0), "r"(0), "r"(fb) : "memory");
      }
    }
  } else if (warp == 5) {
    if (elect_one()) {  // MMA issuer
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ2_BN >> 3) << 17) |
                             ((uint32_t)(OZ_BM >> 4) << 24);
      const auto mma = [&](uint32_t col, uint64_t ad, uint64_t bd, uint32_t acc) {
        asm volatile(
            "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
            ::"r"(tmem + col), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      };
      for (int q = 0; q < NQ; ++q) {
        const int ph = q / KT, kt = q % KT, st = q % OZ2_ST;
        if (ph == 2 && kt == 0) {  // TMEM handed back by the hi epilogue
          mbar_wait(saddr(&tmem_free), 0);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        mbar_wait(saddr(&full[st]), (q / OZ2_ST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a0 = saddr(sm + st * OZ2_STAGE), b0 = a0 + 4 * OZ2_PLANE;
        const uint64_t adb = sdesc_sw64(a0), bdb = sdesc_sw64(b0);
        if (ph == 0) {  // s = 0..3 (A planes 0-3), t = g - s >= 1 (B planes 1-7 at local t - 1)
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2)
#pragma unroll
            for (int g = 4; g < 8; ++g) {
              const int t = g - s2;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t ad = adb + (uint64_t)((s2 * OZ2_PLANE + h * 32) >> 4);
                const uint64_t bd = bdb + (uint64_t)(((t - 1) * OZ2_PLANE + h * 32) >> 4);
                mma((uint32_t)((g - 4) * OZ2_BN), ad, bd, (kt > 0 || s2 > 0 || h > 0) ? 1u : 0u);
              }
            }
        } else if (ph == 1) {  // s = 4..7 (A planes 4-7 at local s - 4), t = g - s in 0..3
#pragma unroll
          for (int s2 = 4; s2 < 8; ++s2)
#pragma unroll
            for (int g = s2; g < 8; ++g) {
              const int t = g - s2;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t ad = adb + (uint64_t)(((s2 - 4) * OZ2_PLANE + h * 32) >> 4);
                const uint64_t bd = bdb + (uint64_t)((t * OZ2_PLANE + h * 32) >> 4);
                mma((uint32_t)((g - 4) * OZ2_BN), ad, bd, 1u);
              }
            }
        } else {  // lo: g = 0..3, s + t = g
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int s2 = 0; s2 <= g; ++s2) {
              const int t = g - s2;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t ad = adb + (uint64_t)((s2 * OZ2_PLANE + h * 32) >> 4);
                const uint64_t bd = bdb + (uint64_t)((t * OZ2_PLANE + h * 32) >> 4);
                mma((uint32_t)(g * OZ2_BN), ad, bd, (kt > 0 || s2 > 0 || h > 0) ? 1u : 0u);
              }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(saddr(&empty[st])));
        if (q == 2 * KT - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(saddr(&done_hi)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(saddr(&done_lo)));
    }
  } else {  // warps 0-3: the two epilogues on their TMEM lane quarters
    mbar_wait(saddr(&done_hi), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    oz2_epilogue<0>(tmem, warp, lane, m0, n0, eu, ex, L, R, N, y);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&tmem_free)) : "memory");
    mbar_wait(saddr(&done_lo), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    oz2_epilogue<1>(tmem, warp, lane, m0, n0, eu, ex, L, R, N, y);
  }
  __syncwarp();  // producer / issuer lanes rejoin their warps
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    TMB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Error(TMB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return (EncodeFn)f;
  }();
  return fn;
}

// 3-D map over digit planes [s][rows][Kp] (uint8), box (64 B of K, box_rows, box_planes), SWIZZLE_64B
CUtensorMap digit_map(int8_t* base, int64_t rows, int64_t Kp, uint32_t box_rows, uint32_t box_planes = OZ_S,
                      uint32_t box_k = OZ_BK) {
  CUtensorMap mp;
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)OZ_S};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(Kp * rows)};
  const cuuint32_t box[3] = {box_k, box_rows, box_planes};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 box_k == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(TMB_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return mp;
}

}  // namespace

void ozaki_cache_slot(Ctx& c, int i, const void* x, DType tx, int64_t L, int64_t K, int64_t R) {
  const int64_t MX = L * R;
  const int64_t Xp = ceil_div(MX, OZ_BN) * OZ_BN, Kp = ceil_div(K, OZ_BK) * OZ_BK;
  Ctx::OzSlot& z = c.ozs[i];
  z = Ctx::OzSlot{};
  z.ex = alloc<int>(c, (size_t)Xp);
  z.sx = alloc<int8_t>(c, (size_t)OZ_S * Xp * Kp);
  z.x = x; z.L = L; z.K = K; z.R = R; z.tx = (int)tx;
}

bool ozaki_enabled() {
  static const bool on = [] {
    const char* s = std::getenv("TMB_OZAKI");  // 0 = DMMA for every contraction
    return !(s && s[0] == '0');
  }();
  return on;
}

void ozaki_ttm(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t R, const double* mat, int64_t N,
               int64_t sMr, int64_t sMk, double* y) {
  // default: the one-pass 128 x 64 tile kernel; TMB_OZ_N128=1 selects the three-pass
  // 128 x 128 variant (bitwise identical; measured 1.11 vs 1.10 ms on the C2 mode-1 pass,
  // tensor pipe ~49 % in both -- the operand port was not the bound)
  static const bool n64 = [] {
    const char* e = std::getenv("TMB_OZ_N128");
    return !(e && e[0] == '1');
  }();
  const int bn = n64 ? OZ_BN : OZ2_BN;
  const int64_t MX = L * R;  // tensor rows
  const int64_t Xp = ceil_div(MX, bn) * bn, Up = ceil_div(N, OZ_BM) * OZ_BM, Kp = ceil_div(K, OZ_BK) * OZ_BK;
  if (K > 65536) throw Error(TMB_EINVAL, "ozaki_ttm: K too large for int32 digit accumulation");
  const size_t mk = c.arena.mark();
  Ctx::OzSlot* slot = nullptr;  // the operand's digit planes from an earlier pass of this solve
  for (auto& z : c.ozs)
    if (z.x == x && z.L == L && z.K == K && z.R == R && z.tx == (int)tx && n64) slot = &z;
  int* ex = slot ? slot->ex : alloc<int>(c, (size_t)Xp);
  int* eu = alloc<int>(c, (size_t)Up);
  int8_t* sx = slot ? slot->sx : alloc<int8_t>(c, (size_t)OZ_S * Xp * Kp);
  int8_t* su = alloc<int8_t>(c, (size_t)OZ_S * Up * Kp);
  // algorithmic work of the fp64-equivalent product: 2 MX N K
  Timed timed(c, TAG_OZAKI, 2.0 * (double)MX * N * K);  // fp64-equivalent flops
  if (slot && slot->valid) {
    // digit planes and row exponents already in place
  } else if (tx == F32 && L % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
    k_oz_rowexp_v4<<<(unsigned)ceil_div(MX, 128), 256, 0, c.stream>>>((const float*)x, L, K, R, ex);
  } else if (L >= 32) {
    if (tx == F32) k_oz_rowexp<float><<<(unsigned)ceil_div(MX, 32), 256, 0, c.stream>>>((const float*)x, L, K, R, ex);
    else k_oz_rowexp<double><<<(unsigned)ceil_div(MX, 32), 256, 0, c.stream>>>((const double*)x, L, K, R, ex);
  } else {
    if (tx == F32)
      k_oz_rowexp<float><<<(unsigned)ceil_div(MX * 32, 256), 256, 0, c.stream>>>((const float*)x, L, K, R, ex);
    else
      k_oz_rowexp<double><<<(unsigned)ceil_div(MX * 32, 256), 256, 0, c.stream>>>((const double*)x, L, K, R, ex);
  }
  if (!(slot && slot->valid)) {
    c.launches++;
    check_launch("k_oz_rowexp");
    dim3 ga((unsigned)ceil_div(Kp, 128), (unsigned)ceil_div(Xp, 32));
    if (tx == F32) k_oz_sliceA<float><<<ga, 256, 0, c.stream>>>((const float*)x, L, K, R, ex, Xp, Kp, sx);
    else k_oz_sliceA<double><<<ga, 256, 0, c.stream>>>((const double*)x, L, K, R, ex, Xp, Kp, sx);
    c.launches++;
    check_launch("k_oz_sliceA");
    if (slot) slot->valid = true;
  }
  k_oz_colexp<<<(unsigned)ceil_div(N * 32, 256), 256, 0, c.stream>>>(mat, K, N, sMr, sMk, eu);
  c.launches++;
  check_launch("k_oz_colexp");
  k_oz_sliceB<<<(unsigned)std::min<int64_t>(ceil_div(Up * Kp, 256), 16LL * c.num_sms), 256, 0, c.stream>>>(
      mat, K, N, sMr, sMk, eu, Up, Kp, su);
  c.launches++;
  check_launch("k_oz_sliceB");
  dim3 grid((unsigned)(Up / OZ_BM), (unsigned)(Xp / bn));
  if (!n64) {
    const CUtensorMap ta4 = digit_map(su, Up, Kp, OZ_BM, 4), tb7 = digit_map(sx, Xp, Kp, OZ2_BN, 7),
                      tb4 = digit_map(sx, Xp, Kp, OZ2_BN, 4);
    const size_t smem = (size_t)OZ2_ST * OZ2_STAGE + 1024;
    set_smem_attr(c, (const void*)k_oz_gemm2, smem);
    k_oz_gemm2<<<grid, OZ2_NT, smem, c.stream>>>(ta4, tb7, tb4, eu, ex, L, R, N, Kp, y);
    c.launches++;
    check_launch("k_oz_gemm2");
  } else {
    // K bytes per stage: 64 (SWIZZLE_64B, 2 x 96 KB stages; default) or 32 (SWIZZLE_32B, 4 x 48 KB:
    // bitwise equal, measured 1.50 vs 1.45 ms for the C2 mode-1 pass -- ring depth is not the bound)
    static const int bkb = [] {
      const char* e = std::getenv("TMB_OZ_BK");
      return e && std::atoi(e) == 32 ? 32 : 64;
    }();
    const CUtensorMap ta = digit_map(su, Up, Kp, OZ_BM, OZ_S, (uint32_t)bkb),
                      tb = digit_map(sx, Xp, Kp, (uint32_t)bn, OZ_S, (uint32_t)bkb);
    const size_t smem = (bkb == 64 ? 2 : 4) * (size_t)OZ_S * (OZ_BM + OZ_BN) * bkb + 1024;
    const void* fn = bkb == 64 ? (const void*)k_oz_gemm<64> : (const void*)k_oz_gemm<32>;
    set_smem_attr(c, fn, smem);
    if (bkb == 64) k_oz_gemm<64><<<grid, OZ_NT, smem, c.stream>>>(ta, tb, eu, ex, L, R, N, Kp, y);
    else k_oz_gemm<32><<<grid, OZ_NT, smem, c.stream>>>(ta, tb, eu, ex, L, R, N, Kp, y);
    c.launches++;
    check_launch("k_oz_gemm");
  }
  c.arena.release(mk);
}

}  // namespace tmb
