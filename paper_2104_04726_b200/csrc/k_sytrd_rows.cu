// Row-partitioned one-stage Householder tridiagonalisation (dsytrd's role in
// eigh, tensor.py:195) -- the production path for 400 < n <= 2048.
//
// Same algorithm and barrier structure as k_sytrd (k_eig.cu: one grid barrier
// per column, rank-2 update of step k fused with the symv of step k+1), but
// with the data partitioned the other way round:
//  * thread t of every block owns rows i = t + 256 u (u < RPT); the pieces of
//    v_k, w_k, v_{k+1} for those rows live in REGISTERS for the whole step,
//    so the fused pass does no shared-memory traffic per element (the column-
//    per-warp kernel needed three 8-byte LDS per element and was bound by it);
//  * block b owns columns j = b mod NB; its 256 threads sweep all rows of an
//    owned column with loads for a batch of columns issued together, and the
//    per-column dot products are reduced with one barrier for all columns;
//  * K = tau/2 p^T v is formed from each thread's own rows (p and v are both
//    row-distributed), so no per-block partial array and no extra gather;
//  * the Householder scalars are computed redundantly by every thread.
// Deterministic: fixed reduction trees, identical in every block.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "tmb_internal.cuh"

namespace cg = cooperative_groups;

namespace tmb {
namespace {


struct RowArgs {
  double* A;
  int64_t n, k_end;
  double* d; double* e; double* tau; double* hv;
  double* pbuf;  // 2 x n: p_k by step parity
  int64_t ld = 0;  // k_sytrd_smem: leading dimension of A and hv (0: n) -- a trailing block of a larger matrix
  int resume = 0;  // k_sytrd_smem: reflector 0 (hv column 0, tau[0]) and d[0], e[0] already computed by
                   // the kernel that ran the earlier steps; A holds rows/columns >= 1 updated through them
  int scribe = 0;  // k_sytrd_smem: block 0 owns no columns (see the kernel)
};

__device__ __forceinline__ double frcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pairwise tree over t[0..M): t[i] += t[i + ceil(M/2)] level by level (for a power
// of two the halving tree; also valid for 12 warps). Result in t[0].
template <int M>
__device__ __forceinline__ void tree_sum(double* t) {
  if constexpr (M > 1) {
    constexpr int H = (M + 1) / 2;
#pragma unroll
    for (int i = 0; i < M - H; ++i) t[i] += t[i + H];
    tree_sum<H>(t);
  }
}

// Block sum, broadcast; fixed order (8 warps). One barrier per call: the warp
// partials alternate between two 8-slot buffers, so a buffer is only rewritten
// after another call's barrier has passed every reader.
// Split form: bsum_put (warp sum -> slot) ... one __syncthreads shared with
// other publications ... bsum_get (fixed-order tree); bitwise equal to bsum.
template <int NW>
__device__ __forceinline__ const double* bsum_put(double v, double* red, int& phase) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* r = red + NW * phase;
  phase ^= 1;
  if (lane == 0) r[w] = v;
  return r;
}

template <int NW>
__device__ __forceinline__ double bsum_get(const double* r) {
  double t[NW];
#pragma unroll
  for (int i = 0; i < NW; i += 2) {
    const double2 q = *reinterpret_cast<const double2*>(r + i);
    t[i] = q.x;
    t[i + 1] = q.y;
  }
  tree_sum<NW>(t);
  return t[0];
}

template <int NW>
__device__ __forceinline__ double bsum(double v, double* red, int& phase) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* r = red + NW * phase;
  phase ^= 1;
  if (lane == 0) r[w] = v;
  __syncthreads();
  double t[NW];
#pragma unroll
  for (int i = 0; i < NW; i += 2) {  // 16-byte broadcast loads: half the LSU instructions
    const double2 q = *reinterpret_cast<const double2*>(r + i);
    t[i] = q.x;
    t[i + 1] = q.y;
  }
  tree_sum<NW>(t);  // pairwise tree: depth log2(NW)
  return t[0];
}

// RPT: rows per thread (n <= 256 RPT); RW_CB: owned columns whose loads are
// issued together (memory-level parallelism vs registers).
template <int RPT, int RW_CB, int RW_THREADS>
__global__ void __launch_bounds__(RW_THREADS, 512 / RW_THREADS) k_sytrd_rows(const RowArgs a) {
  constexpr int NW = RW_THREADS / 32;
  cg::grid_group grid = cg::this_grid();
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NB = gridDim.x, b = blockIdx.x;
  double* A = a.A;
  extern __shared__ double sm[];
  double* vks = sm;            // n: v_k (full, for per-column scalars)
  double* wks = sm + n;        // n: w_k
  double* part = sm + 2 * n;   // NW warps x 64 columns: per-warp partial dots
  double* red = part + NW * 64; // 2 x NW
  int rph = 0;

  double vr[RPT], wr[RPT], nr[RPT];  // v_k, w_k, v_{k+1} on own rows
  // ---- prologue: reflector 0 from column 0 (rows >= 1), every thread redundantly
  double x0[RPT];
  double s2 = 0.0, alpha = 0.0;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t i = tid + (int64_t)RW_THREADS * u;
    x0[u] = (i >= 1 && i < n) ? A[i] : 0.0;
    if (i >= 2 && i < n) s2 = fma(x0[u], x0[u], s2);
  }
  alpha = A[1];
  double xn2 = bsum<NW>(s2, red, rph);
  double tau_k = 0.0, beta = alpha, scale = 0.0;
  if (xn2 > 0.0) {
    const double nrm = sqrt(alpha * alpha + xn2);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau_k = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t i = tid + (int64_t)RW_THREADS * u;
    vr[u] = i == 1 ? 1.0 : (i >= 2 && i < n ? x0[u] * scale : 0.0);
    if (i < n) vks[i] = vr[u];
  }
  if (b == 0) {
    if (tid == 0) { a.d[0] = A[0]; a.e[0] = beta; a.tau[0] = tau_k; }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = tid + (int64_t)RW_THREADS * u;
      if (i < n) a.hv[i] = vr[u];
    }
  }
  __syncthreads();
  // p_0 = tau_0 A v_0 on owned columns j >= 1 (no update yet)
  {
    int q = 0;
    for (int64_t j0 = (b >= 1 ? b : b + NB); j0 < n; j0 += (int64_t)NB * RW_CB, q += RW_CB) {
      double col[RW_CB][RPT];
#pragma unroll
      for (int c = 0; c < RW_CB; ++c)
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t j = j0 + (int64_t)c * NB, i = tid + (int64_t)RW_THREADS * u;
          col[c][u] = (j < n && i >= 1 && i < n) ? A[i + n * j] : 0.0;
        }
#pragma unroll
      for (int c = 0; c < RW_CB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) acc = fma(col[c][u], vr[u], acc);
        acc = wsum(acc);
        if (lane == 0) part[warp * 64 + q + c] = acc;
      }
    }
    __syncthreads();
    if (tid < q) {
      const int64_t j = (b >= 1 ? b : b + NB) + (int64_t)tid * NB;
      if (j < n) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += part[w * 64 + tid];
        a.pbuf[j] = tau_k * s;
      }
    }
  }
  grid.sync();

  for (int64_t k = 0; k + 2 < n && k < a.k_end; ++k) {
    const int buf = (int)(k & 1);
    const double* pb = a.pbuf + buf * n;
    const int64_t c1 = k + 1;
    // ---- gather (one round trip): p_k and column c1 on own rows + the two pivots
    double pp[RPT], xa[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = tid + (int64_t)RW_THREADS * u;
      const bool live = i >= c1 && i < n;
      pp[u] = live ? pb[i] : 0.0;
      xa[u] = live ? A[i + n * c1] : 0.0;
    }
    const double p_c1 = pb[c1], p_k2 = pb[k + 2], a_k2 = A[(k + 2) + n * c1];
    double pv = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) pv = fma(pp[u], vr[u], pv);  // rows < c1 contribute 0
    const double K = 0.5 * tau_k * bsum<NW>(pv, red, rph);
    // ---- w_k and the updated column c1 on own rows
    const double v_c1 = vks[c1], v_k2 = vks[k + 2];
    const double w_c1 = p_c1 - K * v_c1, w_k2 = p_k2 - K * v_k2;
    s2 = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = tid + (int64_t)RW_THREADS * u;
      wr[u] = pp[u] - K * vr[u];
      xa[u] = xa[u] - vr[u] * w_c1 - wr[u] * v_c1;  // x on rows >= c1 (garbage below, masked)
      if (i >= k + 3 && i < n) s2 = fma(xa[u], xa[u], s2);
    }
    if (k + 3 == n) {  // last reflector applied: finish the 2x2 trailing block
      if (b == 0) {
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t i = tid + (int64_t)RW_THREADS * u;
          if (i == n - 2) a.d[n - 2] = xa[u];
          if (i == n - 1) {
            a.e[n - 2] = xa[u];
            a.d[n - 1] = A[(n - 1) + n * (n - 1)] - 2.0 * vr[u] * wr[u];
            a.tau[n - 2] = 0.0;
          }
        }
      }
      break;
    }
    xn2 = bsum<NW>(s2, red, rph);
    // ---- next reflector, every thread redundantly (alpha = x[k+2])
    alpha = a_k2 - v_k2 * w_c1 - w_k2 * v_c1;
    double tau_n = 0.0;
    beta = alpha;
    scale = 0.0;
    if (xn2 > 0.0) {
      const double nrm = sqrt(alpha * alpha + xn2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau_n = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = tid + (int64_t)RW_THREADS * u;
      nr[u] = i == k + 2 ? 1.0 : (i >= k + 3 && i < n ? xa[u] * scale : 0.0);
      if (i >= c1 && i < n) wks[i] = wr[u];
    }
    if (b == 0) {
      if (tid == 0) { a.e[c1] = beta; a.tau[c1] = tau_n; }
      double* h = a.hv + n * c1;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t i = tid + (int64_t)RW_THREADS * u;
        if (i < n) h[i] = nr[u];
        if (i == c1) a.d[c1] = xa[u];
      }
    }
    __syncthreads();  // wks ready (vks holds v_k)
    // ---- fused pass over owned columns j >= k+2: rank-2 update with (v_k, w_k), dot with v_{k+1}
    double* pbn = a.pbuf + (buf ^ 1) * n;
    const int64_t jfirst = b + (int64_t)NB * ((k + 2 - b + NB - 1 > 0 ? (k + 2 - b + NB - 1) : 0) / NB);
    int q = 0;
    for (int64_t j0 = jfirst; j0 < n; j0 += (int64_t)NB * RW_CB, q += RW_CB) {
      double col[RW_CB][RPT];
#pragma unroll
      for (int c = 0; c < RW_CB; ++c)
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t j = j0 + (int64_t)c * NB, i = tid + (int64_t)RW_THREADS * u;
          col[c][u] = (j < n && i >= k + 2 && i < n) ? A[i + n * j] : 0.0;
        }
#pragma unroll
      for (int c = 0; c < RW_CB; ++c) {
        const int64_t j = j0 + (int64_t)c * NB;
        if (j >= n) break;
        const double vj = vks[j], wj = wks[j];
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t i = tid + (int64_t)RW_THREADS * u;
          if (i >= k + 2 && i < n) {
            const double x = col[c][u] - vr[u] * wj - wr[u] * vj;
            A[i + n * j] = x;
            acc = fma(x, nr[u], acc);
          }
        }
        acc = wsum(acc);
        if (lane == 0) part[warp * 64 + q + c] = acc;
      }
    }
    __syncthreads();  // per-warp partials complete; everyone done reading vks/wks
    if (tid < q) {
      const int64_t j = jfirst + (int64_t)tid * NB;
      if (j < n) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += part[w * 64 + tid];
        pbn[j] = tau_n * s;
      }
    }
    // v_k <- v_{k+1}
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = tid + (int64_t)RW_THREADS * u;
      vr[u] = nr[u];
      if (i >= k + 2 && i < n) vks[i] = nr[u];
    }
    tau_k = tau_n;
    grid.sync();
  }
}


// Shared-memory-resident variant (n <= ~1990 on 148 SMs): block b keeps its
// owned columns j = jb + NB q in SHARED memory for the whole reduction, so the
// fused update+symv pass streams shared memory instead of L2 (the L2 variant
// above spends most of a step in dependent L2 round trips). Only what other
// blocks read goes to global: p_{k+1} (pbuf) and the column that becomes the
// next pivot column (k+2), published by its owner during the pass.
// Same arithmetic, in the same order, as k_sytrd_rows (bitwise identical for the
// same block shape; the reduction trees depend on the thread count).
//
// CREG > 0 (register-resident variant): the block's LAST CREG owned columns --
// the ones that stay live longest -- are kept in REGISTERS (thread t holds its
// RPT rows of each), only the earlier ones in shared memory (qsm columns). The
// fused pass is bound by shared-memory bandwidth (one 8-byte load + store per
// element and step); register columns take that traffic away, and once the
// shared-memory columns have retired (k > jb + NB qb) the pass touches no
// memory at all. Same arithmetic and reduction trees per column as CREG = 0.
//
// Measured and removed: a software-pipelined pass (next group's loads issued before the
// current group's arithmetic, each group's shuffle reduction deferred by one group):
// n = 1920 12.3 vs 8.2 ms, n = 1080 4.3 vs 3.7 ms -- the pass is bound by shared-memory /
// MIO throughput (69 % of 128 B/clk with all columns in shared memory), not by its latencies.
//
// UBS: the pass specialised on the block-uniform count ub = k2 / NT of row groups u that are
// dead for EVERY thread (row i = tid + NT u): variant J runs u = J .. RPT-1 as straight-line
// code with NO per-row predicates (only the last u keeps the beyond-the-matrix guard). Rows
// of group u = J that are already dead are processed anyway: they have v = w = 0 (unchanged)
// or are row k+1 (finite junk nobody reads), and v_{k+1} = 0 there, so the dot products are
// unchanged. The predicated form keeps the RPT row predicates in general registers (there are
// 7 predicate registers) and re-tests one per element: as many ISETP as DFMA in the ncu mix.
template <int RPT, int NT, bool PROF, int CREG = 0, int BPS = 512 / NT, int UBS = 0>
__global__ void __launch_bounds__(NT, BPS) k_sytrd_smem(const RowArgs a, int qmax, int qsm, long long* prof) {
  long long t_[10];
#define SM_T(ix) if constexpr (PROF) t_[ix] = clock64();
  constexpr int NW = NT / 32;
  cg::grid_group grid = cg::this_grid();
  const int N = (int)a.n;
  const int64_t n = a.n;
  const int64_t ld = a.ld ? a.ld : a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // scribe mode (TMB_SMEM_SCRIBE=1, off by default: measured no gain, 8.45 vs 8.45 ms at
  // n = 1920): block 0 owns no columns -- it only does the redundant per-step work and the
  // stores of the reflectors / d / e / tau; blocks 1.. share the columns
  const int blk = blockIdx.x;
  const int NB = a.scribe ? (int)gridDim.x - 1 : (int)gridDim.x;  // column-owning blocks
  const int b = a.scribe ? blk - 1 : blk;                         // owner index (-1: the scribe)
  double* A = a.A;
  extern __shared__ double sm[];
  double* cols = sm;                          // qmax x N, column q = jb + NB q
  double* part = cols + ((size_t)qsm * N + 1) / 2 * 2;   // NW x qmax per-warp partial dots (16-B aligned)
  double* red = part + NW * qmax;             // 2 x NW
  double* vo = red + 2 * NW;                  // qmax: v_k at the owned column indices
  double* wo = vo + qmax;                     // qmax: w_k at the owned column indices
  double* piv = wo + qmax;                    // [0] = v_k[k+2]
  int rph = 0;
  const int jb = b < 0 ? N : (b >= 1 ? b : b + NB);  // column 0 is only read (reflector 0)
  const int nown = jb < N ? (N - 1 - jb) / NB + 1 : 0;
  int qi[RPT];                                // slot of row i if i is an owned column index
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int i = tid + NT * u;
    qi[u] = (i >= jb && i < N && (i - jb) % NB == 0) ? (i - jb) / NB : -1;
  }
  // slots [0, qb) live in shared memory, slots qb + r (r < nreg <= CREG) in registers
  const int qb = CREG > 0 ? (nown > CREG ? nown - CREG : 0) : nown;
  const int nreg = nown - qb;
  for (int q = 0; q < qb; ++q) {
    const double* src = A + ld * (jb + (int64_t)NB * q);
    for (int i = tid; i < N; i += NT) cols[q * N + i] = src[i];
  }
  double ar[(CREG > 0 ? CREG : 1) * RPT];
  if constexpr (CREG > 0) {
#pragma unroll
    for (int r = 0; r < CREG; ++r) {
      const double* src = A + ld * (jb + (int64_t)NB * (qb + (r < nreg ? r : 0)));
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = tid + NT * u;
        ar[r * RPT + u] = (r < nreg && i < N) ? src[i] : 0.0;
      }
    }
  }

  double vr[RPT], wr[RPT], nr[RPT];
  double x0[RPT];
  double s2 = 0.0, alpha = 0.0;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int i = tid + NT * u;
    x0[u] = (i >= 1 && i < N) ? A[i] : 0.0;
    if (i >= 2 && i < N) s2 = fma(x0[u], x0[u], s2);
  }
  alpha = A[1];
  double xn2 = bsum<NW>(s2, red, rph);
  double tau_k = 0.0, beta = alpha, scale = 0.0;
  if (xn2 > 0.0) {
    const double nrm = sqrt(alpha * alpha + xn2);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau_k = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int i = tid + NT * u;
    vr[u] = i == 1 ? 1.0 : (i >= 2 && i < N ? x0[u] * scale : 0.0);
    if (qi[u] >= 0) vo[qi[u]] = vr[u];
    if (i == 2) piv[0] = vr[u];
  }
  if (a.resume) {  // continue a reduction: v_0 and tau_0 come from the earlier kernel
    tau_k = a.tau[0];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + NT * u;
      vr[u] = (i >= 1 && i < N) ? a.hv[i] : 0.0;
      if (qi[u] >= 0) vo[qi[u]] = vr[u];
      if (i == 2) piv[0] = vr[u];
    }
  } else if (blk == 0) {
    if (tid == 0) { a.d[0] = A[0]; a.e[0] = beta; a.tau[0] = tau_k; }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + NT * u;
      if (i < N) a.hv[i] = vr[u];
    }
  }
  __syncthreads();
  // p_0 = tau_0 A v_0 on owned columns (no update yet)
  for (int q = 0; q < qb; ++q) {
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + NT * u;
      const double cv = (i >= 1 && i < N) ? cols[q * N + i] : 0.0;
      acc = fma(cv, vr[u], acc);
    }
    acc = wsum(acc);
    if (lane == 0) part[warp * qmax + q] = acc;
  }
  if constexpr (CREG > 0) {
#pragma unroll
    for (int r = 0; r < CREG; ++r) {
      if (r < nreg) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int i = tid + NT * u;
          const double cv = (i >= 1 && i < N) ? ar[r * RPT + u] : 0.0;
          acc = fma(cv, vr[u], acc);
        }
        acc = wsum(acc);
        if (lane == 0) part[warp * qmax + qb + r] = acc;
      }
    }
  }
  __syncthreads();
  if (tid < nown) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += part[w * qmax + tid];
    a.pbuf[jb + (int64_t)NB * tid] = tau_k * s;
  }
  grid.sync();

  int q0 = 0, jq0 = jb;  // first live owned slot and its column index (jb + NB q0 >= k + 2)
  const int qlast_own = ((N - 1 - jb) % NB == 0 && N - 1 >= jb) ? (N - 1 - jb) / NB : -1;
  int64_t k = 0;
  for (; k + 2 < n && k < a.k_end; ++k) {
    SM_T(0);
    const int buf = (int)(k & 1);
    const double* pb = a.pbuf + buf * n;
    const int c1 = (int)k + 1;
    double pp[RPT], xa[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + NT * u;
      const bool live = i >= c1 && i < N;
      pp[u] = live ? pb[i] : 0.0;
      xa[u] = live ? A[i + ld * c1] : 0.0;
    }
    const double p_c1 = pb[c1], p_k2 = pb[k + 2], a_k2 = A[(k + 2) + ld * c1];
    double pv = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) pv = fma(pp[u], vr[u], pv);
    SM_T(1);
    const double K = 0.5 * tau_k * bsum<NW>(pv, red, rph);
    SM_T(2);
    const double v_c1 = 1.0, v_k2 = piv[0];  // v_k[k+1] = 1 by construction
    const double w_c1 = p_c1 - K * v_c1, w_k2 = p_k2 - K * v_k2;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      wr[u] = pp[u] - K * vr[u];
      xa[u] = xa[u] - vr[u] * w_c1 - wr[u] * v_c1;
    }
    if (k + 3 == n) {
      if (blk == 0) {
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int i = tid + NT * u;
          if (i == N - 2) a.d[N - 2] = xa[u];
          if (i == N - 1) {
            a.e[N - 2] = xa[u];
            a.d[N - 1] = A[(n - 1) + ld * (n - 1)] - 2.0 * vr[u] * wr[u];
            a.tau[N - 2] = 0.0;
          }
        }
      }
      break;
    }
    // x is zero at rows < k+1 and >= N already (v_k, w_k and the gathered column are zero
    // there); the two rows that must not count in ||x||^2 -- k+1 (the new diagonal entry,
    // kept in x_c1 by its owner) and k+2 (alpha) -- are zeroed by the ONE thread that holds
    // each, in a rarely taken branch, so the sums below need no per-row predicates (the
    // per-row tests cost ~45 + ~65 instructions per warp and step in the ncu source view)
    static_assert((NT & (NT - 1)) == 0, "row ownership tests assume a power-of-two block");
    const int d1 = c1 - tid, d2 = d1 + 1;
    const bool own1 = d1 >= 0 && (d1 & (NT - 1)) == 0, own2 = d2 >= 0 && (d2 & (NT - 1)) == 0;
    double x_c1 = 0.0;
    if (own1 || own2) {
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = tid + NT * u;
        if (i == c1) { x_c1 = xa[u]; xa[u] = 0.0; }
        if (i == c1 + 1) xa[u] = 0.0;
      }
    }
    s2 = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) s2 = fma(xa[u], xa[u], s2);
    // w_k at the owned indices and the warp partials of ||x||^2 are published
    // behind ONE block barrier (the pass needs wo; every thread then forms
    // ||x||^2 from the partials in bsum's fixed order)
#pragma unroll
    for (int u = 0; u < RPT; ++u)
      if (qi[u] >= 0) wo[qi[u]] = wr[u];
    const double* xr = bsum_put<NW>(s2, red, rph);
    __syncthreads();  // wo + ||x||^2 partials ready
    xn2 = bsum_get<NW>(xr);
    SM_T(3);
    alpha = a_k2 - v_k2 * w_c1 - w_k2 * v_c1;
    double tau_n = 0.0;
    beta = alpha;
    scale = 0.0;
    if (xn2 > 0.0) {
      // reciprocals by rcp.approx + 2 Newton steps (independent, ~1 ulp)
      // instead of two IEEE divisions on the step's serial path
      const double nrm = sqrt(alpha * alpha + xn2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau_n = (beta - alpha) * frcp(beta);
      scale = frcp(alpha - beta);
    }
    SM_T(4);
#pragma unroll
    for (int u = 0; u < RPT; ++u) nr[u] = __fma_rn(xa[u], scale, 0.0);  // + 0.0: no -0 at the zero rows
    if (own2) {
#pragma unroll
      for (int u = 0; u < RPT; ++u)
        if (tid + NT * u == c1 + 1) nr[u] = 1.0;
    }
    if (blk == 0) {
      if (tid == 0) { a.e[c1] = beta; a.tau[c1] = tau_n; }
      if (own1) a.d[c1] = x_c1;
      double* h = a.hv + ld * c1;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = tid + NT * u;
        if (i < N) h[i] = nr[u];
      }
    }
    SM_T(5);
    double* pbn = a.pbuf + (buf ^ 1) * n;
    const int k2 = (int)k + 2;
    // q0 = ceil((k2 - jb) / NB) = number of owned columns below k2, kept incrementally (k2
    // grows by one per step): the integer divisions by the runtime NB sat on the step's
    // serial path (n = 1080: 3.48 -> 3.30 ms, n = 1920: 7.91 -> 7.57 ms without them)
    if (jq0 < k2) { ++q0; jq0 += NB; }
    // Owned live columns, four per iteration: the loads/updates of the four
    // interleave, and their four warp dot products are reduced together with a
    // butterfly reduce-scatter (6 shuffles instead of 20). Shuffles share the
    // MIO pipe with the shared-memory traffic that bounds this pass.
    bool lv[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) lv[u] = tid + NT * u >= k2 && tid + NT * u < N;
    const int qpub = jq0 == k2 ? q0 : -1;            // slot of column k2 if this block owns it
    const int qlast = k2 + 2 == N ? qlast_own : -1;  // slot of column N - 1 before the last step
    // ub: row groups dead for every thread of the block (block-uniform)
    const int ub = k2 / NT;
    const bool padok = tid + NT * (RPT - 1) < N;
    bool ubs_done = false;
    if constexpr (UBS) {
      const bool up = lane & 16, up2 = lane & 8;
      const int cs = (up ? 2 : 0) + (up2 ? 1 : 0);  // column slot this lane's sum belongs to
      auto pass_from = [&](auto jc) {
        constexpr int J = decltype(jc)::value;
        for (int q = q0; q < qb; q += 4) {
          double acc[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            acc[c] = 0.0;
            if (q + c < qb) {
              const double vj = vo[q + c], wj = wo[q + c];
              double* cq = cols + (q + c) * N + tid;
#pragma unroll
              for (int u = J; u < RPT; ++u) {
                if (u < RPT - 1 || padok) {
                  const double xv = cq[NT * u] - vr[u] * wj - wr[u] * vj;
                  cq[NT * u] = xv;
                  acc[c] = fma(xv, nr[u], acc[c]);
                }
              }
            }
          }
          const double r0 = (up ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, up ? acc[0] : acc[2], 16);
          const double r1 = (up ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, up ? acc[1] : acc[3], 16);
          double t = (up2 ? r1 : r0) + __shfl_xor_sync(0xffffffffu, up2 ? r0 : r1, 8);
          t += __shfl_xor_sync(0xffffffffu, t, 4);
          t += __shfl_xor_sync(0xffffffffu, t, 2);
          t += __shfl_xor_sync(0xffffffffu, t, 1);
          if ((lane & 7) == 0 && q + cs < qb) part[warp * qmax + q + cs] = t;
        }
        if constexpr (CREG > 0) {
#pragma unroll
          for (int g = 0; g < CREG; g += 4) {
            if (g < nreg && qb + g + 3 >= q0) {
              double acc[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                acc[c] = 0.0;
                if (g + c < CREG) {
                  const int r = g + c < CREG ? g + c : 0;
                  if (g + c < nreg && qb + g + c >= q0) {
                    const double vj = vo[qb + g + c], wj = wo[qb + g + c];
#pragma unroll
                    for (int u = J; u < RPT; ++u) {  // rows beyond the matrix hold zeros and have v = w = 0
                      const double xv = ar[r * RPT + u] - vr[u] * wj - wr[u] * vj;
                      ar[r * RPT + u] = xv;
                      acc[c] = fma(xv, nr[u], acc[c]);
                    }
                  }
                }
              }
              const double r0 = (up ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, up ? acc[0] : acc[2], 16);
              const double r1 = (up ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, up ? acc[1] : acc[3], 16);
              double t = (up2 ? r1 : r0) + __shfl_xor_sync(0xffffffffu, up2 ? r0 : r1, 8);
              t += __shfl_xor_sync(0xffffffffu, t, 4);
              t += __shfl_xor_sync(0xffffffffu, t, 2);
              t += __shfl_xor_sync(0xffffffffu, t, 1);
              if ((lane & 7) == 0 && g + cs < nreg && qb + g + cs >= q0) part[warp * qmax + qb + g + cs] = t;
            }
          }
        }
      };
      if (N > NT * (RPT - 1) && ub < RPT) {  // only the last row group may reach beyond the matrix
        ubs_done = true;
        switch (ub) {
          case 0: pass_from(std::integral_constant<int, 0>{}); break;
          case 1: pass_from(std::integral_constant<int, (RPT > 1 ? 1 : 0)>{}); break;
          case 2: pass_from(std::integral_constant<int, (RPT > 2 ? 2 : 0)>{}); break;
          case 3: pass_from(std::integral_constant<int, (RPT > 3 ? 3 : 0)>{}); break;
          case 4: pass_from(std::integral_constant<int, (RPT > 4 ? 4 : 0)>{}); break;
          case 5: pass_from(std::integral_constant<int, (RPT > 5 ? 5 : 0)>{}); break;
          case 6: pass_from(std::integral_constant<int, (RPT > 6 ? 6 : 0)>{}); break;
          default: pass_from(std::integral_constant<int, (RPT > 7 ? 7 : 0)>{}); break;
        }
      }
    }
    if (!ubs_done) {
    for (int q = q0; q < qb; q += 4) {
      double acc[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c] = 0.0;
        if (q + c < qb) {
          const double vj = vo[q + c], wj = wo[q + c];
          double* cq = cols + (q + c) * N + tid;
#pragma unroll
          for (int u = 0; u < RPT; ++u) {
            if (lv[u]) {
              const double xv = cq[NT * u] - vr[u] * wj - wr[u] * vj;
              cq[NT * u] = xv;
              acc[c] = fma(xv, nr[u], acc[c]);
            }
          }
        }
      }
      const bool up = lane & 16, up2 = lane & 8;
      const double r0 = (up ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, up ? acc[0] : acc[2], 16);
      const double r1 = (up ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, up ? acc[1] : acc[3], 16);
      double t = (up2 ? r1 : r0) + __shfl_xor_sync(0xffffffffu, up2 ? r0 : r1, 8);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      const int cs = (up ? 2 : 0) + (up2 ? 1 : 0);  // column slot this lane's sum belongs to
      if ((lane & 7) == 0 && q + cs < qb) part[warp * qmax + q + cs] = t;
    }
    if constexpr (CREG > 0) {
      // register-resident columns, four per group (static register indices; the
      // group / column guards are block-uniform)
#pragma unroll
      for (int g = 0; g < CREG; g += 4) {
        if (g < nreg && qb + g + 3 >= q0) {
        double acc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[c] = 0.0;
          if (g + c < CREG) {
            const int r = g + c < CREG ? g + c : 0;
            if (g + c < nreg && qb + g + c >= q0) {
              const double vj = vo[qb + g + c], wj = wo[qb + g + c];
#pragma unroll
              for (int u = 0; u < RPT; ++u) {
                if (lv[u]) {
                  const double xv = ar[r * RPT + u] - vr[u] * wj - wr[u] * vj;
                  ar[r * RPT + u] = xv;
                  acc[c] = fma(xv, nr[u], acc[c]);
                }
              }
            }
          }
        }
        const bool up = lane & 16, up2 = lane & 8;
        const double r0 = (up ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, up ? acc[0] : acc[2], 16);
        const double r1 = (up ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, up ? acc[1] : acc[3], 16);
        double t = (up2 ? r1 : r0) + __shfl_xor_sync(0xffffffffu, up2 ? r0 : r1, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        const int cs = (up ? 2 : 0) + (up2 ? 1 : 0);
        if ((lane & 7) == 0 && g + cs < nreg && qb + g + cs >= q0) part[warp * qmax + qb + g + cs] = t;
        }
      }
    }
    }
    // publish the next pivot column (and, before the last step, the last diagonal)
    if (qpub >= q0 && qpub >= 0 && qpub < nown) {
      double* gq = A + ld * k2;
      if (qpub < qb) {
#pragma unroll
        for (int u = 0; u < RPT; ++u)
          if (lv[u]) gq[tid + NT * u] = cols[qpub * N + tid + NT * u];
      } else if constexpr (CREG > 0) {
        // selects, not an if-chain on the slot: alternative branches with the
        // same body get merged into one with a dynamic (local-memory) index
        const int rp = qpub - qb;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          double xv = ar[u];
#pragma unroll
          for (int r = 1; r < CREG; ++r) xv = rp == r ? ar[r * RPT + u] : xv;
          if (lv[u]) gq[tid + NT * u] = xv;
        }
      }
    }
    if (qlast >= 0 && qlast < nown && tid == (N - 1) % NT) {
      if (qlast < qb) A[(n - 1) + ld * (n - 1)] = cols[qlast * N + N - 1];
      else if constexpr (CREG > 0) {
        const int rl = qlast - qb;
        double xv = 0.0;
#pragma unroll
        for (int r = 0; r < CREG; ++r)
#pragma unroll
          for (int u = 0; u < RPT; ++u) xv = (rl == r && tid + NT * u == N - 1) ? ar[r * RPT + u] : xv;
        A[(n - 1) + ld * (n - 1)] = xv;
      }
    }
    SM_T(6);
    __syncthreads();
    SM_T(7);
    if (tid >= q0 && tid < nown) {
      // the NW warp partials of column tid: all loads first, then a pairwise
      // tree (depth log2 NW instead of an NW-long dependent add chain)
      double t[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) t[w] = part[w * qmax + tid];
      tree_sum<NW>(t);
      pbn[jb + (int64_t)NB * tid] = tau_n * t[0];
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      vr[u] = nr[u];
      if (qi[u] >= 0) vo[qi[u]] = nr[u];
    }
    {  // v_{k+1}[k+3] for the next step, from the one thread that holds row k+3
      const int d3 = d2 + 1;
      if (d3 >= 0 && (d3 & (NT - 1)) == 0) {
#pragma unroll
        for (int u = 0; u < RPT; ++u)
          if (tid + NT * u == c1 + 2) piv[0] = nr[u];
      }
    }
    tau_k = tau_n;
    SM_T(8);
    grid.sync();
    if (PROF && tid == 0 && (blk == 0 || blk == (int)gridDim.x / 2)) {
      SM_T(9);
      long long* r = prof + ((blk ? 1 : 0) * 4 + (int)(4 * k / n)) * 10;
      for (int ph = 0; ph < 9; ++ph) atomicAdd((unsigned long long*)(r + ph), (unsigned long long)(t_[ph + 1] - t_[ph]));
      atomicAdd((unsigned long long*)(r + 9), 1ull);
    }
  }
#undef SM_T
  if (k + 2 < n) {  // stopped at k_end: the trailing block (rows/columns > k) continues from global memory
    for (int q = 0; q < qb; ++q) {
      const int64_t j = jb + (int64_t)NB * q;
      if (j <= k) continue;
      double* dst = A + ld * j;
      for (int i = (int)k + 1 + tid; i < N; i += NT) dst[i] = cols[q * N + i];
    }
    if constexpr (CREG > 0) {
#pragma unroll
      for (int r = 0; r < CREG; ++r) {
        const int64_t j = jb + (int64_t)NB * (qb + r);
        if (r < nreg && j > k) {
          double* dst = A + ld * j;
#pragma unroll
          for (int u = 0; u < RPT; ++u) {
            const int i = tid + NT * u;
            if (i >= (int)k + 1 && i < N) dst[i] = ar[r * RPT + u];
          }
        }
      }
    }
  }
}


}  // namespace

// Shared-memory-resident launch; false if the owned columns do not fit.
// resume < 0: probe only -- returns whether the launch would fit, launches nothing.
bool sytrd_smem(Ctx& c, double* A, int64_t n, int64_t k_end, double* d, double* e, double* tau, double* hv,
                double* pbuf, int64_t ld, int resume) {
  static const int nt_env = [] {
    const char* s = std::getenv("TMB_SMEM_NT");  // A/B: 256 (2 blocks/SM) or 512 (1 block/SM)
    return s ? std::atoi(s) : 0;
  }();
  static const int bps_env = [] {
    const char* s = std::getenv("TMB_SMEM_BPS");  // A/B: blocks per SM
    return s ? std::atoi(s) : 0;
  }();
  static const int creg_env = [] {
    const char* s = std::getenv("TMB_SMEM_CREG");  // A/B: register-resident columns per block (0: none)
    return s ? std::atoi(s) : -1;
  }();
  // default (measured, scripts/gpu_s5_creg.sh): ONE 256-thread block per SM with the last 4
  // owned columns in registers -- n = 1080: 4.11 -> 3.56 ms, n = 1920: 8.45 -> 8.00 ms against
  // the 512-thread blocks (fewer warps shorten every block reduction on the step's serial
  // path; the register columns take the rest). TMB_SMEM_NT=512 restores the old shape.
  const int creg = creg_env >= 0 ? creg_env : 4;
  const int nt = nt_env ? nt_env : 256;
  // (128- and 384-thread blocks measured no better: n = 1920 10.99 / 7.95 ms, n = 1080 3.86 / 3.76 ms)
  const bool regvar = nt == 256 && bps_env != 2;  // one block per SM, up to 255 registers
  const int bps = bps_env ? bps_env : 1;
  static const int nb_env = [] {
    const char* s = std::getenv("TMB_SMEM_NB");  // A/B: grid size (blocks)
    return s ? std::atoi(s) : 0;
  }();
  const int nb = nb_env > 0 ? std::min(nb_env, bps * c.num_sms) : bps * c.num_sms;
  const int rpt = (int)ceil_div(n, nt);
  static const bool rpt4_env = std::getenv("TMB_SMEM_RPT4") != nullptr;  // A/B: 4 rows/thread for n <= 1536
  using KFn = void (*)(RowArgs, int, int, long long*);
  KFn kern = nullptr;
  static const int scribe_env = [] {
    const char* s = std::getenv("TMB_SMEM_SCRIBE");  // A/B: block 0 stores the reflectors and owns no columns
    return s ? std::atoi(s) : -1;
  }();
  const int scribe = scribe_env >= 0 ? (scribe_env != 0) : 0;
  const int qmax = (int)ceil_div(n - 1, nb - scribe);
  static const bool prof_on = std::getenv("TMB_TRD_PROFILE") != nullptr;
#define SMEM_K(R, T) (prof_on ? k_sytrd_smem<R, T, true> : k_sytrd_smem<R, T, false>)
  static const int ubs_env = [] {
    const char* s = std::getenv("TMB_SMEM_UBS");  // A/B: predicate-free pass variants (see the kernel)
    return s ? std::atoi(s) : 1;
  }();
  // measured (scripts/gpu_s5_ubs.sh): the predicate-free variants win only at 8 rows per thread
  // (n = 1920: 7.27 -> 7.17 ms; n = 1080: 3.34 -> 3.40 ms, n = 1500: 5.01 -> 5.09 ms), so only
  // that shape is instantiated with them
#define SMEM_KR(R, T, C)                                                                                           \
  (ubs_env && (R) == 8 ? (prof_on ? k_sytrd_smem<R, T, true, C, 1, ((R) == 8 ? 1 : 0)>                             \
                                  : k_sytrd_smem<R, T, false, C, 1, ((R) == 8 ? 1 : 0)>)                            \
                       : (prof_on ? k_sytrd_smem<R, T, true, C, 1> : k_sytrd_smem<R, T, false, C, 1>))
  int cr = 0;  // register-resident columns of the chosen instantiation
  if (regvar && nt == 256) {
    // (2, 6 and 8 register columns measured no better than 4: n = 1920 8.16 / 8.24 / 9.41 vs 7.98 ms)
    cr = creg >= 4 ? 4 : 0;
#define SMEM_PICK(R) (cr == 4 ? SMEM_KR(R, 256, 4) : SMEM_KR(R, 256, 0))
#define SMEM_PICK4(R) SMEM_PICK(R)
    if (rpt <= 3) { kern = SMEM_PICK4(3); }
    else if (rpt <= 4) { kern = SMEM_PICK4(4); }
    else if (rpt <= 5) { kern = SMEM_PICK(5); }
    else if (rpt <= 6) { kern = SMEM_PICK4(6); }
    else if (rpt <= 7) { kern = SMEM_PICK4(7); }
    else if (rpt <= 8) { kern = SMEM_PICK(8); }
#undef SMEM_PICK
#undef SMEM_PICK4
  } else if (nt == 512) {
    if (rpt <= 2) { kern = SMEM_K(2, 512); }
    else if (rpt <= 3 && !rpt4_env) { kern = SMEM_K(3, 512); }  // n <= 1536 (C2 mode 0)
    else if (rpt <= 4) { kern = SMEM_K(4, 512); }
  } else {
    if (rpt <= 4) { kern = SMEM_K(4, 256); }
    else if (rpt <= 8) { kern = SMEM_K(8, 256); }
  }
#undef SMEM_K
#undef SMEM_KR
  if (!kern) return false;
  const int nw = nt / 32;
  const int qsm = std::max(qmax - cr, 0);  // shared-memory columns per block
  const size_t smem = sizeof(double) * (((size_t)qsm * n + 1) / 2 * 2 + (size_t)nw * qmax + 2 * nw + 2 * qmax + 1);
  if (smem > 227 * 1024) return false;
  set_smem_attr(c, (const void*)kern, std::max<size_t>(smem, 48 * 1024));
  if (blocks_per_sm(c, (const void*)kern, nt, smem) < bps) return false;
  if (resume < 0) return true;
  // TMB_TRD_PROFILE: per-phase clock64 sums (blocks 0 and NB/2, by quarter of the reduction)
  long long* prof = nullptr;
  if (prof_on) {
    prof = alloc<long long>(c, 80);
    TMB_CUDA(cudaMemsetAsync(prof, 0, sizeof(long long) * 80, c.stream));
  }
  RowArgs ra{A, n, k_end, d, e, tau, hv, pbuf, ld, resume, scribe};
  void* args[] = {&ra, (void*)&qmax, (void*)&qsm, &prof};
  TMB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, nb, nt, args, smem, c.stream));
  c.launches++;
  check_launch("k_sytrd_smem");
  if (prof) {
    long long h[80];
    TMB_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    for (int blk = 0; blk < 2; ++blk)
      for (int qtr = 0; qtr < 4; ++qtr) {
        const long long* r = h + (blk * 4 + qtr) * 10;
        if (!r[9]) continue;
        const long long m = r[9];
        std::fprintf(stderr, "sytrd_smem n=%lld blk %d q%d cycles/step: gather %lld K %lld xn2 %lld housemath %lld "
                     "nr+wo+bar %lld pass %lld bar %lld pwrite %lld gridsync %lld\n", (long long)n, blk, qtr,
                     r[0] / m, r[1] / m, r[2] / m, r[3] / m, r[4] / m, r[5] / m, r[6] / m, r[7] / m, r[8] / m);
      }
  }
  return true;
}

// Returns false when n is outside the row-partitioned kernel's range (the
// caller then uses the column-per-warp kernel).
bool sytrd_rows(Ctx& c, double* A, int64_t n, int64_t k_end, double* d, double* e, double* tau, double* hv,
                double* pbuf) {
  if (n > 2048 || n < 3) return false;  // rows per thread <= 8 (256 threads) / 4 (512 threads)
  static const bool smem_off = std::getenv("TMB_SYTRD_L2") != nullptr;  // A/B: force the L2-streaming variant
  // measured (scripts/ab_smem.sh): n=1920 8.8 vs 11.9 ms, n=1080 4.4 vs 5.0 ms,
  // n=500 1.75 vs 1.65 ms (L2 variant keeps small n)
  if (!smem_off && n > 600 && sytrd_smem(c, A, n, k_end, d, e, tau, hv, pbuf, n, 0)) return true;
  static const int cb_env = [] {
    const char* s = std::getenv("TMB_ROWS_CB");  // A/B: columns per load batch
    return s ? std::atoi(s) : 0;
  }();
  static const int nt_env = [] {
    const char* s = std::getenv("TMB_ROWS_NT");  // A/B: 256 or 512 threads per block
    return s ? std::atoi(s) : 0;
  }();
  using KFn = void (*)(RowArgs);
  KFn kern;
  int nt;
  // measured (scripts/ab_rows.sh): 512 threads win only for large n (n=1920:
  // 15.2 vs 16.2 ms; n=1080: 7.3 vs 6.9 ms)
  const bool big_blocks = nt_env == 512 || (nt_env == 0 && n > 1536);
  if (big_blocks) {
    nt = 512;
    const int rpt = (int)ceil_div(n, 512);
    if (rpt <= 2) { kern = cb_env == 1 ? k_sytrd_rows<2, 1, 512> : k_sytrd_rows<2, 2, 512>; }
    else { kern = cb_env == 1 ? k_sytrd_rows<4, 1, 512> : k_sytrd_rows<4, 2, 512>; }
  } else {
    nt = 256;
    const int rpt = (int)ceil_div(n, 256);
    // defaults from scripts/ab_rows.sh: CB 2 / 2 / 1 / 2 for RPT 2 / 4 / 6 / 8
    if (rpt <= 2) { kern = cb_env == 1 ? k_sytrd_rows<2, 1, 256> : k_sytrd_rows<2, 2, 256>; }
    else if (rpt <= 4) { kern = cb_env == 1 ? k_sytrd_rows<4, 1, 256> : k_sytrd_rows<4, 2, 256>; }
    else if (rpt <= 6) { kern = cb_env == 2 ? k_sytrd_rows<6, 2, 256> : k_sytrd_rows<6, 1, 256>; }
    else { kern = cb_env == 1 ? k_sytrd_rows<8, 1, 256> : k_sytrd_rows<8, 2, 256>; }
  }
  const size_t smem = sizeof(double) * (2 * n + (nt / 32) * 64 + 2 * (nt / 32));
  set_smem_attr(c, (const void*)kern, std::max<size_t>(smem, 48 * 1024));
  const int per_sm = blocks_per_sm(c, (const void*)kern, nt, smem);
  if (per_sm < 1) return false;
  // at most 64 owned columns per block (the partial array), ~n/NB per block
  const int64_t need = ceil_div(n, 64);
  const int64_t blocks = std::min<int64_t>((int64_t)per_sm * c.num_sms, std::max<int64_t>(n, 1));
  if (blocks < need) return false;
  RowArgs ra{A, n, k_end, d, e, tau, hv, pbuf};
  void* args[] = {&ra};
  TMB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, (int)blocks, nt, args, smem, c.stream));
  c.launches++;
  check_launch("k_sytrd_rows");
  return true;
}

}  // namespace tmb
