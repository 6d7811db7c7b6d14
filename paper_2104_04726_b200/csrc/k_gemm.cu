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
#include <cstdlib>

#include "tmb_internal.cuh"

namespace tmb {
namespace {

#ifndef TMB_GEMM_ST
#define TMB_GEMM_ST 4
#endif
#ifndef TMB_GEMM_BM
#define TMB_GEMM_BM 64
#endif
// CTA tile BM x 64 x 16; warps of 32x32 (BM/32 along M, 2 along N)
#ifndef TMB_GEMM_BN
#define TMB_GEMM_BN 64
#endif
constexpr int BM = TMB_GEMM_BM, BN = TMB_GEMM_BN, BK = 16, ST = TMB_GEMM_ST, WMW = BM / 32, NT = 32 * WMW * (BN / 32);
constexpr int MINB = 512 / NT;  // resident CTAs per SM the register budget is sized for

template <typename T> struct Pad;
template <> struct Pad<double> { static constexpr int v = 4; };  // 132 = 4 mod 16 (8B banks)
template <> struct Pad<float> { static constexpr int v = 8; };   // 136 = 8 mod 32 (4B banks)

// Shared-memory image of one ROWS x BK operand tile. MF ("rows fast": the
// operand's row index has unit global stride) stores [k][row]; otherwise the
// k index is the contiguous one and the tile is stored [row][k]. Both pads keep
// the DMMA fragment reads (lanes g = row, tig = k) conflict-free and the
// 16-byte cp.async destinations aligned.
template <typename T, bool MF, int ROWS>
struct Tile {
  static constexpr int LD = MF ? ROWS + Pad<T>::v : BK + 4;
  static constexpr int SIZE = MF ? BK * LD : ROWS * LD;
  __device__ static constexpr int at(int row, int k) { return MF ? k * LD + row : row * LD + k; }
};

struct KArgs {
  int64_t M, N, K1, K2;
  int batch, splits;
  int64_t kt_total, kt1;
  const void* A; int64_t sAm, sAk1, sAk2, sAb; int a_vec;
  const void* B; int64_t sBn, sBk1, sBk2, sBb; int b_vec;
  double* C; int64_t sCm, sCn, sCb;
  double alpha, beta;
  double* part;
  int syrk;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero fill: `bytes` (<= BYTES) are read, the rest of the
// destination is zeroed; bytes == 0 reads nothing (ragged tile edges).
template <int BYTES>
__device__ __forceinline__ void cp_async_z(uint32_t s, const void* g, int bytes) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(g), "n"(BYTES), "r"(bytes));
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

// Per-thread copy plan of one operand: V-element chunks (V = 16 B / element
// when the contiguous index is 16-byte aligned, else 1), each thread owning
// NIT chunks at a fixed fast coordinate and a slow coordinate stepping by
// SSTEP -- so a k-tile costs one pointer add per chunk, no index division.
template <typename T, bool MF, int ROWS, int V>
struct Plan {
  static constexpr int FAST = MF ? ROWS : BK;     // extent of the contiguous index
  static constexpr int CPR = FAST / V;             // chunks per slow line
  static constexpr int SSTEP = NT / CPR;           // slow-coordinate step per chunk
  static constexpr int NIT = ROWS * BK / V / NT;
  static_assert(NIT >= 1 && NT % CPR == 0, "tile/thread mismatch");
  int64_t off;    // element offset of chunk 0 relative to the k-tile origin
  int64_t step;   // element offset between consecutive chunks
  int fast, slow0;
  __device__ Plan(int tid, int64_t s_row, int64_t s_k1) {
    fast = (tid % CPR) * V;
    slow0 = tid / CPR;
    const int64_t s_fast = MF ? s_row : s_k1, s_slow = MF ? s_k1 : s_row;
    off = fast * s_fast + slow0 * s_slow;
    step = SSTEP * s_slow;
  }
  // rrem / krem: rows and k left inside the tile (clamped to the tile extents).
  __device__ __forceinline__ void issue(T* dst, const T* src, int rrem, int krem) const {
    const int frem = (MF ? rrem : krem) - fast, srem = MF ? krem : rrem;
    const int nb = (frem >= V ? V : (frem > 0 ? frem : 0)) * (int)sizeof(T);
    const T* g = src + off;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int slow = slow0 + it * SSTEP;
      const bool ok = nb > 0 && slow < srem;
      const int row = MF ? fast : slow, k = MF ? slow : fast;
      cp_async_z<V * sizeof(T)>(smem_u32(dst + Tile<T, MF, ROWS>::at(row, k)), ok ? g + it * step : src,
                                ok ? nb : 0);
    }
  }
};

template <typename TA, typename TB, bool AMF, bool BNF>
__global__ void __launch_bounds__(NT, MINB) k_gemm_dmma(const KArgs p) {
  using TlA = Tile<TA, AMF, BM>;
  using TlB = Tile<TB, BNF, BN>;
  constexpr int VA = 16 / sizeof(TA), VB = 16 / sizeof(TB);
  extern __shared__ __align__(16) unsigned char smem[];
  TA* sA = reinterpret_cast<TA*>(smem);
  TB* sB = reinterpret_cast<TB*>(smem + sizeof(TA) * ST * TlA::SIZE);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp % WMW, wn = warp / WMW;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (p.syrk && n0 + BN <= m0) return;  // tile strictly below the diagonal
  const int b = blockIdx.z % p.batch, split = blockIdx.z / p.batch;
  const int64_t per = (p.kt_total + p.splits - 1) / p.splits;
  const int64_t kb = split * per;
  const int64_t ke = kb + per < p.kt_total ? kb + per : p.kt_total;
  const TA* A = static_cast<const TA*>(p.A) + b * p.sAb + m0 * p.sAm;
  const TB* B = static_cast<const TB*>(p.B) + b * p.sBb + n0 * p.sBn;
  const int arem = (int)(p.M - m0 < BM ? p.M - m0 : BM);
  const int brem = (int)(p.N - n0 < BN ? p.N - n0 : BN);

  const Plan<TA, AMF, BM, VA> pav(tid, p.sAm, p.sAk1);
  const Plan<TA, AMF, BM, 1> pas(tid, p.sAm, p.sAk1);
  const Plan<TB, BNF, BN, VB> pbv(tid, p.sBn, p.sBk1);
  const Plan<TB, BNF, BN, 1> pbs(tid, p.sBn, p.sBk1);

  // k-tile cursor of the next load: (k1 offset, slab index), advanced without division
  int64_t lk1 = (kb % p.kt1) * BK, lk2 = kb / p.kt1;
  auto load = [&](int stage) {
    const int krem = (int)(p.K1 - lk1 < BK ? p.K1 - lk1 : BK);
    const TA* ga = A + lk1 * p.sAk1 + lk2 * p.sAk2;
    const TB* gb = B + lk1 * p.sBk1 + lk2 * p.sBk2;
    if (p.a_vec) pav.issue(sA + stage * TlA::SIZE, ga, arem, krem);
    else pas.issue(sA + stage * TlA::SIZE, ga, arem, krem);
    if (p.b_vec) pbv.issue(sB + stage * TlB::SIZE, gb, brem, krem);
    else pbs.issue(sB + stage * TlB::SIZE, gb, brem, krem);
    lk1 += BK;
    if (lk1 >= p.K1) { lk1 = 0; ++lk2; }
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
    if (kb + s < ke) load(s);
    cp_commit();
  }
  int stage = 0;
  for (int64_t kt = kb; kt < ke; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < ke) load(stage == 0 ? ST - 1 : stage - 1);
    cp_commit();
    const TA* cA = sA + stage * TlA::SIZE;
    const TB* cB = sB + stage * TlB::SIZE;
    stage = stage + 1 == ST ? 0 : stage + 1;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      double af[2][4], bf[4][2];
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        const int mb = wm * 32 + ii * 16 + g;
        af[ii][0] = (double)cA[TlA::at(mb, kk + tig)];
        af[ii][1] = (double)cA[TlA::at(mb + 8, kk + tig)];
        af[ii][2] = (double)cA[TlA::at(mb, kk + tig + 4)];
        af[ii][3] = (double)cA[TlA::at(mb + 8, kk + tig + 4)];
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int nb = wn * 32 + jj * 8 + g;
        bf[jj][0] = (double)cB[TlB::at(nb, kk + tig)];
        bf[jj][1] = (double)cB[TlB::at(nb, kk + tig + 4)];
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

template <typename TA, typename TB, bool AMF, bool BNF>
void launch_t(Ctx& c, const KArgs& a, dim3 grid) {
  const size_t smem = (size_t)ST * (Tile<TA, AMF, BM>::SIZE * sizeof(TA) + Tile<TB, BNF, BN>::SIZE * sizeof(TB));
  set_smem_attr(c, (const void*)k_gemm_dmma<TA, TB, AMF, BNF>, smem);
  k_gemm_dmma<TA, TB, AMF, BNF><<<grid, NT, smem, c.stream>>>(a);
  c.launches++;
  check_launch("k_gemm_dmma");
}

template <typename TA, typename TB>
void launch_l(Ctx& c, const KArgs& a, dim3 grid, bool amf, bool bnf) {
  if (amf && bnf) launch_t<TA, TB, true, true>(c, a, grid);
  else if (amf) launch_t<TA, TB, true, false>(c, a, grid);
  else if (bnf) launch_t<TA, TB, false, true>(c, a, grid);
  else launch_t<TA, TB, false, false>(c, a, grid);
}

// 16-byte chunks along the contiguous index need the base and every other
// stride to be multiples of the chunk (in elements).
bool vec_ok(const void* base, int elem, int64_t s_other1, int64_t s_other2, int64_t s_batch) {
  const int64_t v = 16 / elem;
  return reinterpret_cast<uintptr_t>(base) % 16 == 0 && s_other1 % v == 0 && s_other2 % v == 0 &&
         s_batch % v == 0;
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
  const bool amf = (d.sAm == 1) ? true : (d.sAk1 != 1);
  const bool bnf = (d.sBn == 1) ? true : (d.sBk1 != 1);
  const int ea = d.ta == F64 ? 8 : 4, eb = d.tb == F64 ? 8 : 4;
  a.a_vec = (amf ? d.sAm == 1 : d.sAk1 == 1) &&
            vec_ok(d.A, ea, amf ? d.sAk1 : d.sAm, d.K2 > 1 ? d.sAk2 : 0, d.batch > 1 ? d.sAb : 0);
  a.b_vec = (bnf ? d.sBn == 1 : d.sBk1 == 1) &&
            vec_ok(d.B, eb, bnf ? d.sBk1 : d.sBn, d.K2 > 1 ? d.sBk2 : 0, d.batch > 1 ? d.sBb : 0);
  a.C = d.C; a.sCm = d.sCm; a.sCn = d.sCn; a.sCb = d.sCb;
  a.alpha = d.alpha; a.beta = d.beta; a.syrk = d.syrk_upper ? 1 : 0;
  const int64_t tn = ceil_div(d.N, BN), tm = ceil_div(d.M, BM);
  int64_t tiles = tn * tm * d.batch;
  if (d.syrk_upper) tiles = (tiles + tn * d.batch) / 2;
  int splits = d.splits;
  if (splits <= 0) {
    static const int policy = [] {
      const char* s = std::getenv("TMB_GEMM_SPLITS");  // A/B: 0 = fill the resident slots, 1 = 2 CTAs per SM
      return s ? std::atoi(s) : 0;
    }();
    splits = 1;
    if (policy == 1) {
      const int64_t want = 2LL * c.num_sms;
      if (tiles < want && a.kt_total >= 8) {
        splits = (int)std::min<int64_t>(ceil_div(want, tiles), a.kt_total / 4);
        splits = std::max(1, std::min(splits, 64));
      }
    } else {
      // split K only as far as one wave of resident CTAs (MINB per SM) holds: a
      // partial second wave (e.g. 306 CTAs at 2 per SM for the C2 mode-0 Gram)
      // leaves most of the DMMA pipes idle for its duration
      const int64_t slots = (int64_t)MINB * c.num_sms;
      if (tiles < slots && a.kt_total >= 8) {
        splits = (int)std::min<int64_t>(slots / tiles, a.kt_total / 4);
        splits = std::max(1, std::min(splits, 64));
      }
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
  if (d.ta == F64 && d.tb == F64) launch_l<double, double>(c, a, grid, amf, bnf);
  else if (d.ta == F32 && d.tb == F64) launch_l<float, double>(c, a, grid, amf, bnf);
  else if (d.ta == F64 && d.tb == F32) launch_l<double, float>(c, a, grid, amf, bnf);
  else launch_l<float, float>(c, a, grid, amf, bnf);
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
