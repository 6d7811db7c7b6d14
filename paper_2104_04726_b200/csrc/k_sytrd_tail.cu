// Cluster-resident tail of the Householder tridiagonalisation (k_eig.cu).
//
// The grid-wide kernel pays one grid barrier (~1.2 us) plus several L2 round
// trips per column, which is wasteful once the trailing block is small. Here a
// single thread-block cluster (16 CTAs, one per SM, non-portable size; 8 if 16
// is refused) holds the whole trailing m x m block in distributed shared memory
// (column c of the block lives in CTA c mod CL), exchanges p_j / partial sums /
// the next column through DSMEM and synchronises with ONE cluster barrier per
// column. It continues the same algorithm from step K0 (v_{K0}, tau_{K0} in
// hv/tau, A's trailing block updated through step K0-1), or starts from
// scratch (K0 = 0), so small matrices never touch the grid kernel.
#include <cooperative_groups.h>

#include <map>
#include <mutex>

#include "tmb_internal.cuh"

namespace cg = cooperative_groups;

namespace tmb {
namespace {

constexpr int TAIL_THREADS = 512;

struct TailArgs {
  double* A;       // n x n, column-major (trailing block read once)
  int64_t n, K0;
  double* d; double* e; double* tau; double* hv;
};

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum broadcast to all threads: warp partials -> warp 0 shuffle tree ->
// red[32]. Fixed order, identical in every CTA; one LDS per thread instead of
// every thread looping over all warp partials.
__device__ __forceinline__ double bsum(double v, double* red) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    const double x = wsum(lane < nw ? red[lane] : 0.0);
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  return red[32];
}

template <int CL>
__global__ void __launch_bounds__(TAIL_THREADS, 1) k_sytrd_tail(const TailArgs a) {
  static_assert((CL & (CL - 1)) == 0, "cluster size must be a power of two");
  constexpr int SH = CL == 16 ? 4 : (CL == 8 ? 3 : (CL == 4 ? 2 : 1));
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = bd >> 5;
  const int64_t n = a.n, base = a.K0 + 1, m = n - base;  // local index = global - base
  const int64_t nown = (m + CL - 1) / CL;                // columns per CTA (max)
  extern __shared__ double sm[];
  double* cols = sm;                        // nown x m: owned local column c = r + CL*q at cols + q*m
  double* vk = cols + nown * m;             // m (local rows)
  double* wk = vk + m;
  double* vn = wk + m;
  double* pb = vn + m;                      // 2 x nown (p_j of owned columns, by step parity)
  double* part = pb + 2 * nown;             // 2 (partial sum p.v over owned columns)
  double* red = part + 2;                   // 33
  double* sc = red + 33;                    // 8
  double* A = a.A;

  // ---- load owned columns of the trailing block (rows >= base)
  for (int64_t q = 0; q < nown; ++q) {
    const int64_t c = r + (int64_t)CL * q;
    if (c >= m) break;
    const double* src = A + (base + c) * n + base;
    for (int64_t i = tid; i < m; i += bd) cols[q * m + i] = src[i];
  }
  // ---- reflector v_{K0}: given (hv/tau) or computed from column K0 when K0 == 0
  double tau_k;
  if (a.K0 == 0) {
    for (int64_t i = tid; i < m; i += bd) vn[i] = A[base + i];  // column 0, rows >= 1
    __syncthreads();
    double s = 0.0;
    for (int64_t i = 1 + tid; i < m; i += bd) s = fma(vn[i], vn[i], s);
    const double xn2 = bsum(s, red);
    if (tid == 0) {
      const double alpha = vn[0];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (xn2 > 0.0) {
        const double nrm = sqrt(alpha * alpha + xn2);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      sc[0] = t; sc[1] = beta; sc[2] = scale;
    }
    __syncthreads();
    tau_k = sc[0];
    for (int64_t i = tid; i < m; i += bd) vk[i] = i == 0 ? 1.0 : vn[i] * sc[2];
    __syncthreads();
    if (r == 0) {
      if (tid == 0) { a.d[0] = A[0]; a.e[0] = sc[1]; a.tau[0] = tau_k; }
      for (int64_t i = tid; i < n; i += bd) a.hv[i] = i >= 1 ? vk[i - 1] : 0.0;
    }
  } else {
    const double* h = a.hv + n * a.K0;
    for (int64_t i = tid; i < m; i += bd) vk[i] = h[base + i];
    tau_k = a.tau[a.K0];
  }
  __syncthreads();
  // ---- p_{K0} = tau A22 v over owned columns (rows >= base, i.e. local >= 0)
  {
    double wpart = 0.0;
    for (int64_t q = warp; q < nown; q += nw) {
      const int64_t c = r + (int64_t)CL * q;
      if (c >= m) break;
      const double* col = cols + q * m;
      double acc = 0.0;
      for (int64_t i = lane; i < m; i += 32) acc = fma(col[i], vk[i], acc);
      const double p = tau_k * wsum(acc);
      if (lane == 0) pb[q] = p;  // parity 0 buffer
      wpart = fma(p, vk[c], wpart);
    }
    const double s = bsum(lane == 0 ? wpart : 0.0, red);
    if (tid == 0) part[0] = s;
  }
  cl.sync();

  for (int64_t k = a.K0; k + 2 < n; ++k) {
    const int buf = (int)((k - a.K0) & 1);
    const int64_t lk = k + 1 - base;  // local index of row/column k+1 (c1)
    // ---- K = tau/2 sum_r part_r (DSMEM, fixed rank order)
    if (warp == 0) {  // one DSMEM round trip: lane rr loads rank rr's partial
      const double pr = lane < CL ? cl.map_shared_rank(part, lane)[buf] : 0.0;
      const double s = wsum(pr);
      if (lane == 0) sc[3] = 0.5 * tau_k * s;
    }
    __syncthreads();
    const double K = sc[3];
    // ---- w = p - K v (p_j from its owner's smem) and x = updated column c1
    for (int64_t i = lk + tid; i < m; i += bd) {
      const double* opb = cl.map_shared_rank(pb, (int)(i & (CL - 1)));
      wk[i] = opb[buf * nown + (i >> SH)] - K * vk[i];
    }
    __syncthreads();
    if (k + 3 == n) {  // last reflector applied: finish the 2x2 trailing block
      if (r == 0 && tid == 0) {
        const int64_t i2 = n - 2 - base, i3 = n - 1 - base;
        const double* c2 = cl.map_shared_rank(cols, (int)(i2 & (CL - 1))) + (i2 >> SH) * m;
        const double* c3 = cl.map_shared_rank(cols, (int)(i3 & (CL - 1))) + (i3 >> SH) * m;
        a.d[n - 2] = c2[i2] - 2.0 * vk[i2] * wk[i2];
        a.e[n - 2] = c2[i3] - vk[i3] * wk[i2] - wk[i3] * vk[i2];
        a.d[n - 1] = c3[i3] - 2.0 * vk[i3] * wk[i3];
        a.tau[n - 2] = 0.0;
      }
      break;
    }
    const double vj = vk[lk], wj = wk[lk];
    const double* c1col = cl.map_shared_rank(cols, (int)(lk & (CL - 1))) + (lk >> SH) * m;
    double s2 = 0.0;
    for (int64_t i = lk + tid; i < m; i += bd) {
      const double x = c1col[i] - vk[i] * wj - wk[i] * vj;
      if (i == lk) sc[4] = x; else vn[i] = x;
      if (i >= lk + 2) s2 = fma(x, x, s2);
    }
    const double xn2 = bsum(s2, red);
    if (tid == 0) {
      const double alpha = vn[lk + 1];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (xn2 > 0.0) {
        const double nrm = sqrt(alpha * alpha + xn2);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      sc[0] = t; sc[1] = beta; sc[2] = scale;
    }
    __syncthreads();
    const double tau_n = sc[0], scale = sc[2];
    for (int64_t i = lk + 2 + tid; i < m; i += bd) vn[i] *= scale;
    if (tid == 0) vn[lk + 1] = 1.0;
    __syncthreads();
    if (r == 0) {
      const int64_t c1 = k + 1;
      if (tid == 0) { a.d[c1] = sc[4]; a.e[c1] = sc[1]; a.tau[c1] = tau_n; }
      double* h = a.hv + n * c1;
      for (int64_t i = tid; i < n; i += bd) h[i] = (i >= k + 2) ? vn[i - base] : 0.0;
    }
    // ---- fused pass over owned columns j >= k+2 (local >= lk+1)
    double wpart = 0.0;
    const int nb2 = buf ^ 1;
    for (int64_t q = warp; q < nown; q += nw) {
      const int64_t c = r + (int64_t)CL * q;
      if (c >= m) break;
      if (c < lk + 1) continue;
      double* col = cols + q * m;
      const double vjj = vk[c], wjj = wk[c];
      double acc0 = 0.0, acc1 = 0.0;
      int64_t i = lk + 1 + lane;
      for (; i + 32 < m; i += 64) {
        const double x0 = col[i] - vk[i] * wjj - wk[i] * vjj;
        const double x1 = col[i + 32] - vk[i + 32] * wjj - wk[i + 32] * vjj;
        col[i] = x0;
        col[i + 32] = x1;
        acc0 = fma(x0, vn[i], acc0);
        acc1 = fma(x1, vn[i + 32], acc1);
      }
      if (i < m) {
        const double x0 = col[i] - vk[i] * wjj - wk[i] * vjj;
        col[i] = x0;
        acc0 = fma(x0, vn[i], acc0);
      }
      const double p = tau_n * wsum(acc0 + acc1);
      if (lane == 0) pb[nb2 * nown + q] = p;
      wpart = fma(p, vn[c], wpart);
    }
    const double sp = bsum(lane == 0 ? wpart : 0.0, red);
    if (tid == 0) part[nb2] = sp;
    double* t = vk; vk = vn; vn = t;
    tau_k = tau_n;
    cl.sync();
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

struct TailCfg { int cl = 0; int64_t max_m = 0; const void* fn = nullptr; };

TailCfg tail_config_compute(Ctx& c) {
  TailCfg cfg;
  int smem_optin = 0;
  TMB_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
  for (int cl : {16, 8}) {
    const void* fn = cl == 16 ? (const void*)k_sytrd_tail<16> : (const void*)k_sytrd_tail<8>;
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
    if (cl > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cl);
    lc.blockDim = dim3(TAIL_THREADS);
    lc.dynamicSmemBytes = smem_optin;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cl; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    lc.attrs = &at;
    lc.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &lc) == cudaSuccess && nclusters >= 1) {
      // largest m with nown*m + 3m + 2*nown + 42 doubles in smem_optin
      int64_t best = 0;
      for (int64_t mm = 64; mm < 4096; ++mm) {
        const int64_t nown = (mm + cl - 1) / cl;
        if ((nown * mm + 3 * mm + 2 * nown + 48) * 8 <= smem_optin) best = mm; else break;
      }
      cfg.fn = fn;
      cfg.cl = cl;
      cfg.max_m = best;
      return cfg;
    }
    cudaGetLastError();
  }
  return cfg;
}

// per device (cluster attributes and occupancy are per device context), thread-safe
TailCfg tail_config(Ctx& c) {
  static std::mutex mu;
  static std::map<int, TailCfg> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(c.device);
  if (it != cache.end()) return it->second;
  const TailCfg cfg = tail_config_compute(c);
  cache[c.device] = cfg;
  return cfg;
}

}  // namespace

int64_t sytrd_tail_capacity(Ctx& c) { return tail_config(c).max_m; }

void sytrd_tail(Ctx& c, double* A, int64_t n, int64_t K0, double* d, double* e, double* tau, double* hv) {
  const TailCfg cfg = tail_config(c);
  const int64_t m = n - K0 - 1;
  if (cfg.cl == 0 || m > cfg.max_m) throw Error(TMB_EINVAL, "sytrd_tail: trailing block too large for the cluster");
  const int64_t nown = (m + cfg.cl - 1) / cfg.cl;
  const size_t smem = sizeof(double) * (nown * m + 3 * m + 2 * nown + 48);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(cfg.cl);
  lc.blockDim = dim3(TAIL_THREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = c.stream;
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = cfg.cl; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  lc.attrs = &at;
  lc.numAttrs = 1;
  TailArgs ta{A, n, K0, d, e, tau, hv};
  void* args[] = {&ta};
  TMB_CUDA(cudaLaunchKernelExC(&lc, cfg.fn, args));
  c.launches++;
  check_launch("k_sytrd_tail");
}

}  // namespace tmb
