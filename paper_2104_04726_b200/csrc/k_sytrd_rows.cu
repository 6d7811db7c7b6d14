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

#include "tmb_internal.cuh"

namespace cg = cooperative_groups;

namespace tmb {
namespace {


struct RowArgs {
  double* A;
  int64_t n, k_end;
  double* d; double* e; double* tau; double* hv;
  double* pbuf;  // 2 x n: p_k by step parity
};

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum, broadcast; fixed order (8 warps). One barrier per call: the warp
// partials alternate between two 8-slot buffers, so a buffer is only rewritten
// after another call's barrier has passed every reader.
template <int NW>
__device__ __forceinline__ double bsum(double v, double* red, int& phase) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* r = red + NW * phase;
  phase ^= 1;
  if (lane == 0) r[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) s += r[i];
  return s;
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

struct RowsInfo { int blocks = 0; int64_t n = -1; };

}  // namespace

// Returns false when n is outside the row-partitioned kernel's range (the
// caller then uses the column-per-warp kernel).
bool sytrd_rows(Ctx& c, double* A, int64_t n, int64_t k_end, double* d, double* e, double* tau, double* hv,
                double* pbuf) {
  if (n > 2048 || n < 3) return false;  // rows per thread <= 8 (256 threads) / 4 (512 threads)
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
  int slot, nt;
  // measured (scripts/ab_rows.sh): 512 threads win only for large n (n=1920:
  // 15.2 vs 16.2 ms; n=1080: 7.3 vs 6.9 ms)
  const bool big_blocks = nt_env == 512 || (nt_env == 0 && n > 1536);
  if (big_blocks) {
    nt = 512;
    const int rpt = (int)ceil_div(n, 512);
    if (rpt <= 2) { kern = cb_env == 1 ? k_sytrd_rows<2, 1, 512> : k_sytrd_rows<2, 2, 512>; slot = 4; }
    else { kern = cb_env == 1 ? k_sytrd_rows<4, 1, 512> : k_sytrd_rows<4, 2, 512>; slot = 5; }
  } else {
    nt = 256;
    const int rpt = (int)ceil_div(n, 256);
    // defaults from scripts/ab_rows.sh: CB 2 / 2 / 1 / 2 for RPT 2 / 4 / 6 / 8
    if (rpt <= 2) { kern = cb_env == 1 ? k_sytrd_rows<2, 1, 256> : k_sytrd_rows<2, 2, 256>; slot = 0; }
    else if (rpt <= 4) { kern = cb_env == 1 ? k_sytrd_rows<4, 1, 256> : k_sytrd_rows<4, 2, 256>; slot = 1; }
    else if (rpt <= 6) { kern = cb_env == 2 ? k_sytrd_rows<6, 2, 256> : k_sytrd_rows<6, 1, 256>; slot = 2; }
    else { kern = cb_env == 1 ? k_sytrd_rows<8, 1, 256> : k_sytrd_rows<8, 2, 256>; slot = 3; }
  }
  const size_t smem = sizeof(double) * (2 * n + (nt / 32) * 64 + 2 * (nt / 32));
  static RowsInfo info[6];
  if (info[slot].n != n) {
    TMB_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(smem, 48 * 1024)));
    int per_sm = 0;
    TMB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kern, nt, smem));
    if (per_sm < 1) return false;
    // at most 64 owned columns per block (the partial array), ~n/NB per block
    const int64_t need = ceil_div(n, 64);
    int64_t blocks = std::min<int64_t>((int64_t)per_sm * c.num_sms, std::max<int64_t>(n, 1));
    if (blocks < need) return false;
    info[slot].blocks = (int)blocks;
    info[slot].n = n;
  }
  RowArgs ra{A, n, k_end, d, e, tau, hv, pbuf};
  void* args[] = {&ra};
  TMB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, info[slot].blocks, nt, args, smem, c.stream));
  c.launches++;
  check_launch("k_sytrd_rows");
  return true;
}

}  // namespace tmb
