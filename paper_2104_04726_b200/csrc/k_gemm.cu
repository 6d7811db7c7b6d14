// FP64 GEMM on the Blackwell DMMA pipe (mma.sync m16n8k8 f64), the contraction
// engine behind every TTM (tensor.py:111-123), Gram (tensor.py:176-180) and the
// eigen-solver GEMMs.
//
// Why DMMA and not tcgen05: the fit used for trace/best-of/convergence
// (tucker.py:174-191, 379-393) is 1 - sqrt(|t|^2 - |core|^2)/|t|, which
// amplifies relative core error by |t|/resid (~100x at fit 0.99); fp32-class
// intermediates move the fit by ~1e-6 (measured) and the Gram
// eigengaps sit at ~1e-9 lambda_1. tcgen05 has no f64 kind,
// so the contractions run on DMMA, which on B200 measures 37.1 TFLOP/s
// (profiles/r01_probe_peaks.txt), at parity with cuBLAS DGEMM (35.5).
//
// Generic strided operands let every mode-n product / mode-n Gram of an
// F-order tensor run without materialising an unfolding: A(m, k1, k2) and
// B(k1, k2, n) with a two-level inner index (k2 = the slab index of the
// modes after n). Split-K partials are reduced in a fixed order (deterministic,
// no atomics).
#include "tmb_internal.cuh"

namespace tmb {
namespace {

constexpr int BM = 128, BN = 64, BK = 16, ST = 3, NT = 256;

template <typename T> struct Pad;
template <> struct Pad<double> { static constexpr int v = 4; };  // 132 = 4 mod 16 (8B banks)
template <> struct Pad<float> { static constexpr int v = 8; };   // 136 = 8 mod 32 (4B banks)

struct KArgs {
  int64_t M, N, K1, K2;
  int batch, splits;
  int64_t kt_total, kt1;
  const void* A; int64_t sAm, sAk1, sAk2, sAb; int a_mfast;
  const void* B; int64_t sBn, sBk1, sBk2, sBb; int b_nfast;
  double* C; int64_t sCm, sCn, sCb;
  double alpha, beta;
  double* part;
  int syrk;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int BYTES>
__device__ __forceinline__ void cp_async_z(uint32_t s, const void* g, bool valid) {
  int sz = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(g), "n"(BYTES), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(NT, 2) k_gemm_dmma(const KArgs p) {
  constexpr int LDA = BM + Pad<TA>::v, LDB = BN + Pad<TB>::v;
  extern __shared__ __align__(16) unsigned char smem[];
  TA* sA = reinterpret_cast<TA*>(smem);
  TB* sB = reinterpret_cast<TB*>(smem + sizeof(TA) * ST * BK * LDA);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (p.syrk && n0 + BN <= m0) return;  // tile strictly below the diagonal
  const int b = blockIdx.z % p.batch, split = blockIdx.z / p.batch;
  const int64_t per = (p.kt_total + p.splits - 1) / p.splits;
  const int64_t kb = split * per;
  const int64_t ke = kb + per < p.kt_total ? kb + per : p.kt_total;
  const TA* A = static_cast<const TA*>(p.A) + b * p.sAb;
  const TB* B = static_cast<const TB*>(p.B) + b * p.sBb;

  auto load = [&](int stage, int64_t kt) {
    const int64_t k2 = kt / p.kt1, k1b = (kt % p.kt1) * BK;
    TA* dA = sA + stage * BK * LDA;
    TB* dB = sB + stage * BK * LDB;
#pragma unroll
    for (int it = 0; it < BM * BK / NT; ++it) {
      const int e = tid + it * NT;
      int m, k;
      if (p.a_mfast) { m = e % BM; k = e / BM; } else { k = e % BK; m = e / BK; }
      const int64_t gm = m0 + m, gk = k1b + k;
      const bool v = gm < p.M && gk < p.K1;
      const TA* src = v ? A + gm * p.sAm + gk * p.sAk1 + k2 * p.sAk2 : A;
      cp_async_z<sizeof(TA)>(smem_u32(dA + k * LDA + m), src, v);
    }
#pragma unroll
    for (int it = 0; it < BN * BK / NT; ++it) {
      const int e = tid + it * NT;
      int n, k;
      if (p.b_nfast) { n = e % BN; k = e / BN; } else { k = e % BK; n = e / BK; }
      const int64_t gn = n0 + n, gk = k1b + k;
      const bool v = gn < p.N && gk < p.K1;
      const TB* src = v ? B + gn * p.sBn + gk * p.sBk1 + k2 * p.sBk2 : B;
      cp_async_z<sizeof(TB)>(smem_u32(dB + k * LDB + n), src, v);
    }
  };

  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (kb + s < ke) load(s, kb + s);
    cp_commit();
  }
  for (int64_t kt = kb; kt < ke; ++kt) {
    const int i = (int)(kt - kb);
    cp_wait<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < ke) load((i + ST - 1) % ST, kt + ST - 1);
    cp_commit();
    const TA* cA = sA + (i % ST) * BK * LDA;
    const TB* cB = sB + (i % ST) * BK * LDB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      double af[2][4], bf[4][2];
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        const int mb = wm * 32 + ii * 16 + g;
        af[ii][0] = (double)cA[(kk + tig) * LDA + mb];
        af[ii][1] = (double)cA[(kk + tig) * LDA + mb + 8];
        af[ii][2] = (double)cA[(kk + tig + 4) * LDA + mb];
        af[ii][3] = (double)cA[(kk + tig + 4) * LDA + mb + 8];
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int nb = wn * 32 + jj * 8 + g;
        bf[jj][0] = (double)cB[(kk + tig) * LDB + nb];
        bf[jj][1] = (double)cB[(kk + tig + 4) * LDB + nb];
      }
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) dmma(acc[ii][jj], af[ii], bf[jj]);
    }
  }
  cp_wait<0>();

#pragma unroll
  for (int ii = 0; ii < 2; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t row = m0 + wm * 32 + ii * 16 + g + ((r & 2) ? 8 : 0);
        const int64_t col = n0 + wn * 32 + jj * 8 + 2 * tig + (r & 1);
        if (row >= p.M || col >= p.N) continue;
        const double v = acc[ii][jj][r];
        if (p.splits > 1) {
          p.part[((int64_t)(split * p.batch + b) * p.M + row) * p.N + col] = v;
        } else {
          double* cp = p.C + b * p.sCb + row * p.sCm + col * p.sCn;
          *cp = p.beta != 0.0 ? p.alpha * v + p.beta * *cp : p.alpha * v;
        }
      }
}

__global__ void k_splitk_reduce(const KArgs p) {
  const int64_t total = (int64_t)p.batch * p.M * p.N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = e % p.N, row = (e / p.N) % p.M, b = e / (p.N * p.M);
    if (p.syrk && col < row) continue;
    double s = 0.0;
    for (int sp = 0; sp < p.splits; ++sp) s += p.part[((int64_t)(sp * p.batch + b) * p.M + row) * p.N + col];
    double* cp = p.C + b * p.sCb + row * p.sCm + col * p.sCn;
    *cp = p.beta != 0.0 ? p.alpha * s + p.beta * *cp : p.alpha * s;
  }
}

__global__ void k_mirror(double* g, int64_t n, int batch, int64_t sb) {
  const int64_t total = (int64_t)batch * n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = (e / n) % n, b = e / (n * n);
    if (i > j) g[b * sb + i + n * j] = g[b * sb + j + n * i];  // lower <- upper
  }
}

template <typename TA, typename TB>
void launch_t(Ctx& c, const KArgs& a, dim3 grid) {
  constexpr int LDA = BM + Pad<TA>::v, LDB = BN + Pad<TB>::v;
  const size_t smem = (size_t)ST * BK * (LDA * sizeof(TA) + LDB * sizeof(TB));
  static bool attr = false;
  if (!attr) {
    TMB_CUDA(cudaFuncSetAttribute(k_gemm_dmma<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  k_gemm_dmma<TA, TB><<<grid, NT, smem, c.stream>>>(a);
  c.launches++;
  check_launch("k_gemm_dmma");
}

}  // namespace

void gemm(Ctx& c, const GemmDesc& d0) {
  GemmDesc d = d0;
  if (d.M <= 0 || d.N <= 0 || d.batch <= 0) return;
  if (!d.syrk_upper && d.N > d.M) {  // keep the long side on the 128-row tile dimension
    std::swap(d.M, d.N);
    std::swap(d.A, d.B);
    std::swap(d.ta, d.tb);
    std::swap(d.sAm, d.sBn);
    std::swap(d.sAk1, d.sBk1);
    std::swap(d.sAk2, d.sBk2);
    std::swap(d.sAb, d.sBb);
    std::swap(d.sCm, d.sCn);
  }
  KArgs a{};
  a.M = d.M; a.N = d.N; a.K1 = d.K1; a.K2 = d.K1 > 0 ? d.K2 : 0;
  a.batch = d.batch;
  a.kt1 = ceil_div(d.K1, BK);
  a.kt_total = a.kt1 * a.K2;
  a.A = d.A; a.sAm = d.sAm; a.sAk1 = d.sAk1; a.sAk2 = d.sAk2; a.sAb = d.sAb;
  a.B = d.B; a.sBn = d.sBn; a.sBk1 = d.sBk1; a.sBk2 = d.sBk2; a.sBb = d.sBb;
  a.a_mfast = (d.sAm == 1) ? 1 : (d.sAk1 == 1 ? 0 : 1);
  a.b_nfast = (d.sBn == 1) ? 1 : (d.sBk1 == 1 ? 0 : 1);
  a.C = d.C; a.sCm = d.sCm; a.sCn = d.sCn; a.sCb = d.sCb;
  a.alpha = d.alpha; a.beta = d.beta; a.syrk = d.syrk_upper ? 1 : 0;
  const int64_t tn = ceil_div(d.N, BN), tm = ceil_div(d.M, BM);
  int64_t tiles = tn * tm * d.batch;
  if (d.syrk_upper) tiles = (tiles + tn * d.batch) / 2;
  int splits = d.splits;
  if (splits <= 0) {
    splits = 1;
    const int64_t want = 2LL * c.num_sms;
    if (tiles < want && a.kt_total >= 8) {
      splits = (int)std::min<int64_t>(ceil_div(want, tiles), a.kt_total / 4);
      splits = std::max(1, std::min(splits, 64));
    }
  }
  if ((int64_t)splits * d.batch > 65535) splits = std::max<int64_t>(1, 65535 / d.batch);
  a.splits = splits;
  if (splits > 1) a.part = alloc<double>(c, (size_t)splits * d.batch * d.M * d.N);
  if (tm > 65535) throw Error(TMB_EINVAL, "gemm: M too large for the tile grid");
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)(d.batch * splits));
  // algorithmic flops: 2mnk per product, s(s+1)K for a SYRK
  const double kk = (double)d.K1 * (double)d.K2 * d.batch;
  const double work = d.syrk_upper ? (double)d.M * (d.M + 1) * kk : 2.0 * d.M * d.N * kk;
  Timed timed(c, c.gemm_tag, work);
  if (d.ta == F64 && d.tb == F64) launch_t<double, double>(c, a, grid);
  else if (d.ta == F32 && d.tb == F64) launch_t<float, double>(c, a, grid);
  else if (d.ta == F64 && d.tb == F32) launch_t<double, float>(c, a, grid);
  else launch_t<float, float>(c, a, grid);
  if (splits > 1) {
    const int64_t total = (int64_t)d.batch * d.M * d.N;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8LL * c.num_sms);
    k_splitk_reduce<<<blocks, 256, 0, c.stream>>>(a);
    c.launches++;
    check_launch("k_splitk_reduce");
  }
}

void mirror_upper(Ctx& c, double* g, int64_t n, int batch, int64_t sb) {
  const int64_t total = (int64_t)batch * n * n;
  if (total == 0) return;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 8LL * c.num_sms);
  k_mirror<<<blocks, 256, 0, c.stream>>>(g, n, batch, sb);
  c.launches++;
  check_launch("k_mirror");
}

}  // namespace tmb
