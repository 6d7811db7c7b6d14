// Two-stage tridiagonalisation for eigh (tensor.py:195) of the large Grams
// (the default for n > 4600: C5's n = 7680), where the one-stage reduction
// streams the trailing matrix from HBM / L2 once per column.
//
//  stage 1 (sy2sb): dense -> band of half-bandwidth SBR_B. Panel p (columns
//    p0 .. p0+31) is QR-factorised below the band by ONE thread-block cluster
//    (the panel rows split over the cluster's CTAs in shared memory, two
//    cluster all-reduces per column through DSMEM), then the trailing matrix
//    gets the two-sided compact-WY update A22 <- Q^T A22 Q as DMMA GEMMs:
//      X = A22 (V T),  M = V^T X,  W = X - V (T^T M) / 2,  A22 -= V W^T + W V^T
//    (LAPACK's dsytrd blocked update, restated for a band target). The
//    reflectors land in the one-stage layout (column c of hv = reflector of
//    column c, zero above its first row), so the compact-WY back-transformation
//    of the one-stage path applies them unchanged.
//  stage 2 (sb2st): band -> tridiagonal by one-column-at-a-time bulge chasing
//    (Lang's algorithm as in LAPACK dsytrd_sb2st). Task (s, j) = sweep s at
//    position j touches only rows [s+1+jb, s+1+(j+1)b) in lower band storage
//    (2b diagonals: the band + the bulge), so the rows are partitioned over a
//    cluster's CTAs in shared memory and each task runs on the CTA owning its
//    first row, one warp per task. Dependencies: (s, j) after (s, j-1) (its
//    reflector, kept in registers or passed to the next CTA through a DSMEM
//    mailbox) and after (s-1, j+1) (progress counters in shared memory,
//    release/acquire at cluster scope). The reflectors are not stored: the
//    eigenvectors of the band matrix come from inverse iteration on the band
//    (k_band_invit below), so only stage 1's reflectors are back-applied.
//
// Accuracy: Householder reductions throughout (backward stable, the dsytrd
// class); the eigenvalues of T are those of G to eps ||G||.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <set>

#include "tmb_internal.cuh"

namespace cg = cooperative_groups;

namespace tmb {
namespace {

#define LAUNCHED(name) do { c.launches++; check_launch(name); } while (0)

constexpr int SB = SBR_B;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// ------------------------------------------------------------------ stage 1: panel QR
// One thread per panel row, the row's 32 entries in registers: the column loop
// is unrolled so every register index is static, and only the columns right of
// the current one are touched (an unblocked Householder pass re-reading the
// panel from shared memory each column was shared-memory-bandwidth bound).
constexpr int PQ_NT = 512, PQ_NW = PQ_NT / 32;

struct PanelArgs {
  double* A;
  int64_t n, p0;
  double* hv;
  double* tau;
};

// Values val_0 = x^2, val_t = (t > i ? x * row[t] : 0) for 0 < t < 32 -> lane l
// of every warp holds the warp sum of val_l (butterfly reduce-scatter: 31
// shuffles; the first stage forms its operands on the fly so only 16 partials
// are ever live next to the 32 row registers).
__device__ __forceinline__ double rs_row(const double (&row)[SB], double x, int i, int lane) {
  double v[16];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const double a0 = t == 0 ? x * x : (t > i ? x * row[t] : 0.0);
      const double a1 = t + 16 > i ? x * row[t + 16] : 0.0;
      const double send = up ? a0 : a1, keep = up ? a1 : a0;
      v[t] = keep + __shfl_xor_sync(FULL, send, 16);
    }
  }
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int t = 0; t < o; ++t) {
      const double send = up ? v[t] : v[t + o];
      const double keep = up ? v[t + o] : v[t];
      v[t] = keep + __shfl_xor_sync(FULL, send, o);
    }
  }
  return v[0];
}

// Cluster all-reduce of NV <= 64 CTA partials already in xb (this CTA's slot):
// one cluster barrier, then NV threads add the CS partials in rank order (the
// same bits in every CTA) into out.
template <int CS>
__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, double* xb, int nv, double* out) {
  if constexpr (CS > 1) {
    cl.sync();
    const int t = threadIdx.x;
    if (t < nv) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < CS; ++q) s += cl.map_shared_rank(xb, q)[t];
      out[t] = s;
    }
  } else {
    __syncthreads();
    if ((int)threadIdx.x < nv) out[threadIdx.x] = xb[threadIdx.x];
  }
  __syncthreads();
}

template <int CS>
__global__ void __launch_bounds__(PQ_NT, 1) k_panel_qr(const PanelArgs a) {
  __shared__ double xb[2 * 64], red[PQ_NW * 32], bc[64];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = CS > 1 ? (int)cl.block_rank() : 0;
  const int64_t n = a.n, p0 = a.p0, r0 = p0 + SB;
  const int m = (int)(n - r0);
  const int RB = (m + CS - 1) / CS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = rank * RB + tid;  // panel row of this thread
  const bool has = tid < RB && g < m;
  // row[t] = P[g][i + t] for the current column i: the row shifts left by one
  // after every column, so all register indices stay static without unrolling
  // the column loop (the unrolled version was instruction-fetch bound).
  double row[SB];
#pragma unroll
  for (int t = 0; t < SB; ++t) row[t] = has ? a.A[(r0 + g) + n * (p0 + t)] : 0.0;
  const int nref = min(m - 1, SB);
  int par = 0;
  // One cluster all-reduce per column: with x = column i below the diagonal,
  //   [0] = |x|^2, [t >= 1] = sum_g x_g P[g][i+t] (unscaled), [32 + t] = P[i][i+t],
  // so w_t = sum_g v_g P[g][i+t] = P[i][i+t] + [t] / (alpha - beta) (v_i = 1,
  // v_g = x_g / (alpha - beta) below) is formed after the reduction.
  for (int i = 0; i < nref; ++i) {
    const double x = (has && g > i) ? row[0] : 0.0;
    const double ws = rs_row(row, x, 0, lane);
    red[warp * 32 + lane] = ws;
    double* xs = xb + par * 64;
    if (has && g == i) {
#pragma unroll
      for (int t = 0; t < SB; ++t) xs[32 + t] = row[t];
    }
    __syncthreads();
    if (tid < SB) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
      for (int w = 0; w < PQ_NW; w += 4) {
        t0 += red[w * 32 + tid];
        t1 += red[(w + 1) * 32 + tid];
        t2 += red[(w + 2) * 32 + tid];
        t3 += red[(w + 3) * 32 + tid];
      }
      xs[tid] = (t0 + t1) + (t2 + t3);
    } else if (tid < 64 && !(i >= rank * RB && i < rank * RB + RB)) {
      xs[tid] = 0.0;  // no pivot row on this CTA
    }
    cluster_sum<CS>(cl, xs, 64, bc);
    par ^= 1;
    const double xn2 = bc[0], alpha = bc[32];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    const double vg = (has && g > i) ? x * scale : ((has && g == i) ? 1.0 : 0.0);
    const double tv = -vg * tau;
#pragma unroll
    for (int t = 1; t < SB; ++t) row[t] = fma(tv, fma(scale, bc[t], bc[32 + t]), row[t]);
    if (has && g >= i) a.hv[(r0 + g) + n * (p0 + i)] = vg;
    if (has && g == i) {  // row i of R is final
      a.A[(r0 + g) + n * (p0 + i)] = beta;
#pragma unroll
      for (int t = 1; t < SB; ++t)
        if (t < SB - i) a.A[(r0 + g) + n * (p0 + i + t)] = row[t];
    }
    if (rank == 0 && tid == 0) a.tau[p0 + i] = tau;
#pragma unroll
    for (int t = 0; t + 1 < SB; ++t) row[t] = row[t + 1];
    row[SB - 1] = 0.0;
  }
  if (rank == 0 && tid < SB && tid >= nref) a.tau[p0 + tid] = 0.0;
  // rows >= nref (only when m - 1 < SB): their remaining R entries
  if (has && g >= nref && nref < SB)
#pragma unroll
    for (int t = 0; t < SB; ++t)
      if (t < SB - nref && g <= nref + t) a.A[(r0 + g) + n * (p0 + nref + t)] = row[t];
  if constexpr (CS > 1) cl.sync();  // no CTA exits while a peer may read its exchange slots
}

// dlarft (forward, columnwise) for one 32-reflector panel from S = V^T V:
// T(r, i) = -tau_i sum_{r <= c < i} T(r, c) S(c, i). Thread r owns row r of T
// in registers, so the rows proceed independently (no block barriers).
__global__ void __launch_bounds__(SB) k_larft32(const double* __restrict__ S, const double* __restrict__ tau,
                                                double* __restrict__ T) {
  __shared__ double sS[SB * SB], st[SB];
  const int r = threadIdx.x;
  for (int e = r; e < SB * SB; e += SB) sS[e] = S[e];
  st[r] = tau[r];
  __syncthreads();
  double tr[SB];
#pragma unroll
  for (int i = 0; i < SB; ++i) {
    double v = 0.0;
    if (i == r) {
      v = st[i];
    } else if (i > r) {
      double s = 0.0;
#pragma unroll
      for (int cc = 0; cc < i; ++cc)
        if (cc >= r) s = fma(tr[cc], sS[cc + SB * i], s);
      v = -st[i] * s;
    }
    tr[i] = v;
  }
#pragma unroll
  for (int i = 0; i < SB; ++i) T[r + SB * i] = tr[i];
}

// W = X - V (T^T M) / 2 for the m panel rows; writes [V | W | V] (m x 96, ld ldo)
// so the trailing update A22 -= V W^T + W V^T is one GEMM with plain strides.
__global__ void __launch_bounds__(256) k_sbr_w(const double* __restrict__ X, const double* __restrict__ V, int64_t ldv,
                                               const double* __restrict__ M, const double* __restrict__ T, int64_t m,
                                               double* __restrict__ VWV, int64_t ldo) {
  __shared__ double sZ[SB * SB], sM[SB * SB], sT[SB * SB];
  const int tid = threadIdx.x;
  for (int e = tid; e < SB * SB; e += 256) { sM[e] = M[e]; sT[e] = T[e]; }
  __syncthreads();
  for (int e = tid; e < SB * SB; e += 256) {  // Z = T^T M (column-major)
    const int r = e % SB, cc = e / SB;
    double s = 0.0;
    for (int k = 0; k < SB; ++k) s = fma(sT[k + SB * r], sM[k + SB * cc], s);
    sZ[e] = s;
  }
  __syncthreads();
  const int64_t rows_per = 256 / SB;
  const int cc = tid % SB;
  for (int64_t r = (int64_t)blockIdx.x * rows_per + tid / SB; r < m; r += (int64_t)gridDim.x * rows_per) {
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < SB; ++k) s = fma(V[r + ldv * k], sZ[k + SB * cc], s);
    const double v = V[r + ldv * cc];
    VWV[r + ldo * cc] = v;
    VWV[r + ldo * (SB + cc)] = fma(-0.5, s, X[r + m * cc]);
    VWV[r + ldo * (2 * SB + cc)] = v;
  }
}

// Full band rows (|c - r| <= b) of the symmetric A into n x (2b+1): band[r][c - r + b].
__global__ void k_band_rows(const double* __restrict__ A, int64_t n, double* __restrict__ band) {
  constexpr int W = 2 * SB + 1;
  const int64_t total = n * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / W, cc = r + (e % W) - SB;
    double v = 0.0;
    if (cc >= 0 && cc < n) v = r >= cc ? A[r + n * cc] : A[cc + n * r];
    band[e] = v;
  }
}

// ------------------------------------------------------------------ stage 2: bulge chasing
constexpr int S2_W = 8;            // worker warps per CTA (one task each)
constexpr int S2_NS = 32;          // progress / mailbox slots (sweep mod S2_NS)
constexpr int S2_LDL = 2 * SB;     // lower band row: offsets 0 .. 2b-1 (stride 64: the diagonal walks at
                                   // stride 65 are bank-conflict free, 65 made them 2-way)

struct S2Args {
  const double* band;
  int n, R, RS;
  double* spill;
  double* d;
  double* e;
  long long* prof;  // diagnostics (TMB_S2_PROF): per warp [wait cycles, task cycles, tasks]
};

// Progress counters: cluster scope only where producer and consumer sit on
// different CTAs (a cluster-scope release compiles to MEMBAR.ALL.GPU and a
// cluster-scope acquire to an L1 invalidation -- microseconds per task when
// used for every task); the CTA-local hand-offs use CTA scope.
__device__ __forceinline__ unsigned ld_acq_cl(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acq_cta(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void red_max_rel_cl(unsigned* p, unsigned v) {
  asm volatile("red.release.cluster.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_max_rel_cta(unsigned* p, unsigned v) {
  asm volatile("red.release.cta.shared.max.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned tag(int s, int cnt) { return (unsigned)s * 256u + (unsigned)cnt; }

// Householder of the lane-distributed x (x_0 = alpha on lane 0, lanes >= m hold 0):
// H x = beta e_0, H = I - tau v v^T, v_0 = 1 (dlarfg).
__device__ __forceinline__ void house_warp(double x, int lane, double& v, double& tau, double& beta) {
  const double s2 = wsum(lane >= 1 ? x * x : 0.0);
  const double alpha = __shfl_sync(FULL, x, 0);
  if (s2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    v = lane == 0 ? 1.0 : 0.0;
    return;
  }
  beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
  tau = (beta - alpha) / beta;
  v = lane == 0 ? 1.0 : x * (1.0 / (alpha - beta));
}

// 32 broadcast doubles from shared memory into registers (16-byte loads), so
// the compiler can issue them all before a phase's stores (with the loads
// interleaved with stores to the band rows it cannot hoist them: possible alias)
__device__ __forceinline__ void bcast32(const double* src, double (&r)[SB]) {
#pragma unroll
  for (int t = 0; t < SB; t += 2) {
    const double2 q = *reinterpret_cast<const double2*>(src + t);
    r[t] = q.x;
    r[t + 1] = q.y;
  }
}

// Rows q0 .. q0+m-1 of a task in at most two runs of consecutive rows at stride
// S2_LDL: rows [0, h) at base, rows [h, m) at base2 (the next CTA's shared memory
// over DSMEM, or the global spill rows). Lanes >= m are inactive (the last block
// of a sweep).
template <bool SEG, bool PART, bool PROF>
__device__ __forceinline__ void s2_task_fast(double* base, double* base2, int h, int m_, int j, int lane, double vp,
                                             double taup, double* vs, double* ws, double* zs, double& v, double& tau,
                                             long long* ph) {
  auto row = [&](int i) -> double* {
    if constexpr (SEG) return i < h ? base + i * S2_LDL : base2 + (i - h) * S2_LDL;
    return base + i * S2_LDL;
  };
  const int m = PART ? m_ : SB;  // PART: a short last block (lanes >= m inactive)
  const bool act = !PART || lane < m;
  double* rp = row(act ? lane : 0);
  double beta;
  long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // TMB_S2_PROF phase clocks
  if constexpr (PROF) c0 = c1 = c2 = c3 = clock64();
  if (j == 0) {
    const double x = act ? rp[1 + lane] : 0.0;  // column s, rows q0 + lane
    house_warp(x, lane, v, tau, beta);
    if (act) rp[1 + lane] = lane == 0 ? beta : 0.0;
  } else {
    double brow[SB];  // B[lane][jj] = L[q0+lane][SB+lane-jj]
    double* bp = rp + SB + lane;
#pragma unroll
    for (int jj = 0; jj < SB; ++jj) brow[jj] = act ? bp[-jj] : 0.0;
    vs[lane] = vp;
    __syncwarp();
    double b32[SB];
    bcast32(vs, b32);
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int jj = 0; jj < SB; jj += 2) {
      y0 = fma(brow[jj], b32[jj], y0);
      y1 = fma(brow[jj + 1], b32[jj + 1], y1);
    }
    const double ty = taup * (y0 + y1);
#pragma unroll
    for (int jj = 0; jj < SB; ++jj) {
      brow[jj] = fma(-ty, b32[jj], brow[jj]);
      if (act) bp[-jj] = brow[jj];
    }
    if constexpr (PROF) c1 = clock64();
    house_warp(brow[0], lane, v, tau, beta);
    if constexpr (PROF) c2 = clock64();
    ws[lane] = v;
    __syncwarp();
    bcast32(ws, b32);
    // z_lane = sum_i v_i B[i][lane] = sum_i v_i L[q0+i][SB+i-lane]: column walk
    double z0 = 0.0, z1 = 0.0;
#pragma unroll
    for (int i = 0; i < SB; i += 2) {
      if (i < m) z0 = fma(b32[i], row(i)[SB + i - lane], z0);
      if (i + 1 < m) z1 = fma(b32[i + 1], row(i + 1)[SB + i + 1 - lane], z1);
    }
    zs[lane] = tau * (z0 + z1);
    __syncwarp();
    bcast32(zs, b32);
    if (act) {
      bp[0] = lane == 0 ? beta : 0.0;
#pragma unroll
      for (int jj = 1; jj < SB; ++jj) bp[-jj] = fma(-v, b32[jj], brow[jj]);
    }
  }
  __syncwarp();
  if constexpr (PROF) c3 = clock64();
  // D: the lane's full symmetric row; D[lane][c] = L[q0+lane][lane-c] (c <= lane)
  // or L[q0+c][c-lane] = rp[(c - lane) * (S2_LDL + 1)] (c > lane)
  double drow[SB];
  const double* lp = rp + lane;
#pragma unroll
  for (int cc = 0; cc < SB; ++cc) {
    const double* ad = cc <= lane ? lp - cc : row(cc) + (cc - lane);
    drow[cc] = (act && cc < m) ? *ad : 0.0;
  }
  vs[lane] = v;
  __syncwarp();
  double v32[SB];
  bcast32(vs, v32);
  double p0 = 0.0, p1 = 0.0;
#pragma unroll
  for (int cc = 0; cc < SB; cc += 2) {
    p0 = fma(drow[cc], v32[cc], p0);
    p1 = fma(drow[cc + 1], v32[cc + 1], p1);
  }
  const double p = tau * (p0 + p1);
  const double K = 0.5 * tau * wsum(p * v);
  const double w = fma(-K, v, p);
  ws[lane] = w;
  __syncwarp();
  double w32[SB];
  bcast32(ws, w32);
  double* up = rp + lane;
  if (act) {
#pragma unroll
    for (int cc = 0; cc < SB; ++cc)
      if (cc <= lane) up[-cc] = fma(-v, w32[cc], fma(-w, v32[cc], drow[cc]));
  }
  __syncwarp();
  if (PROF && j > 0) {
    const long long c4 = clock64();
    ph[0] += c1 - c0; ph[1] += c2 - c1; ph[2] += c3 - c2; ph[3] += c4 - c3; ph[4] += 1;
  }
}

// Rows are split into NG = CS * RPC ranges of R rows. RPC = 1 (default): CTA c owns
// range c. RPC = 2 (TMB_S2_MIRROR=1, 16-CTA cluster): CTA c owns ranges c and
// 2CS-1-c, a top and the mirrored bottom one, each served by half of its warps --
// row r is touched by ~r/b tasks, so contiguous ranges give the last CTA twice the
// average task count; the mirrored pairs balance it but measured slower (sb2st()).
template <int CS, int RPC, bool PROF>
__global__ void __launch_bounds__(S2_W * 32, 1) k_sb2st(const S2Args a) {
  constexpr int NG = CS * RPC;       // ranges
  constexpr int WP = S2_W / RPC;     // warps per range (slot)
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int cr = CS > 1 ? (int)cl.block_rank() : 0;
  const int n = a.n, R = a.R, RS = a.RS;  // R: rows per range; RS: rows of this CTA in shared memory
  double* rows = sm;                                    // RS x S2_LDL (slot 0's rows, then slot 1's)
  double* hbox = rows + (size_t)RS * S2_LDL;            // RPC x S2_NS x 33 (v, tau) mailboxes
  double* scr = hbox + RPC * S2_NS * 33;                // per warp: vs, ws, zs (3 x 32)
  unsigned* lprog = reinterpret_cast<unsigned*>(scr + S2_W * 96);  // RPC x S2_NS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SPILL = RPC * R - RS;                       // spill rows per CTA
  auto owner = [](int g) { return RPC == 1 || g < CS ? g : 2 * CS - 1 - g; };
  auto slot = [](int g) { return RPC == 1 || g < CS ? 0 : 1; };
  // row r of range g (owned by CTA owner(g), slot slot(g)) given that CTA's rows base
  auto rowp_g = [&](int r, int g, double* base) -> double* {
    const int li = slot(g) * R + (r - g * R);
    if (li < RS) return base + (size_t)li * S2_LDL;
    return a.spill + ((size_t)owner(g) * SPILL + (li - RS)) * S2_LDL;
  };
  for (int sl = 0; sl < RPC; ++sl) {
    const int g = sl == 0 ? cr : 2 * CS - 1 - cr;
    const int glo = g * R, ghi = min(n, glo + R);
    for (int e = tid; e < max(0, ghi - glo) * S2_LDL; e += S2_W * 32) {
      const int r = glo + e / S2_LDL, o = e % S2_LDL;
      double v = 0.0;
      if (o <= SB && r - o >= 0) v = a.band[(size_t)r * (2 * SB + 1) + (SB - o)];
      rowp_g(r, g, rows)[o] = v;
    }
  }
  for (int e = tid; e < RPC * S2_NS; e += S2_W * 32) lprog[e] = 0u;
  if constexpr (CS > 1) cl.sync(); else __syncthreads();
  // this warp's range and its neighbours
  const int sl = warp / WP, wl = warp % WP;
  const int g = sl == 0 ? cr : 2 * CS - 1 - cr;
  const int lo = g * R, hi = min(n, lo + R);
  auto cta_ptr = [&](auto* p, int c) {
    if constexpr (CS > 1) return c == cr ? p : cl.map_shared_rank(p, c);
    else return p;
  };
  double* rows_nx = rows;
  double* hbox_nx = nullptr;
  unsigned* lp_nx = nullptr;
  unsigned* lp_pv = nullptr;
  if (g + 1 < NG) {
    rows_nx = cta_ptr(rows, owner(g + 1));
    hbox_nx = cta_ptr(hbox, owner(g + 1)) + slot(g + 1) * S2_NS * 33;
    lp_nx = cta_ptr(lprog, owner(g + 1)) + slot(g + 1) * S2_NS;
  }
  if (g > 0) lp_pv = cta_ptr(lprog, owner(g - 1)) + slot(g - 1) * S2_NS;
  double* my_hbox = hbox + sl * S2_NS * 33;
  unsigned* my_lp = lprog + sl * S2_NS;
  auto wait_for = [&](int s, int cnt, bool remote) {
    const unsigned want = tag(s, cnt);
    const unsigned* p = my_lp + (s % S2_NS);
    if (remote) {
      while (ld_acq_cl(p) < want) __nanosleep(64);
    } else {
      while (ld_acq_cta(p) < want) __nanosleep(20);
    }
  };
  double* vs = scr + warp * 96;
  double* ws = vs + 32;
  double* zs = vs + 64;
  long long pw = 0, pt = 0, pn = 0;
  long long ph[5] = {0, 0, 0, 0, 0};
  // the first run of a task's rows: this range's shared rows, then its spill rows
  const int li0 = slot(g) * R;                                  // local index of row lo
  const int lsm = li0 >= RS ? lo : lo + min(RS - li0, hi - lo);  // end of the range's shared rows
  for (int s = wl; s <= n - 3; s += WP) {
    if (s + 1 >= hi) break;
    const int jst = lo > s + 1 ? (lo - s - 1 + SB - 1) / SB : 0;
    if (s + 1 + jst * SB >= hi) continue;
    double vp = 0.0, taup = 0.0;
    if (jst > 0) {  // reflector of (s, jst - 1) from the previous range
      const long long t0 = PROF ? clock64() : 0;
      wait_for(s, jst, true);
      if constexpr (PROF) pw += clock64() - t0;
      vp = my_hbox[(s % S2_NS) * 33 + lane];
      taup = my_hbox[(s % S2_NS) * 33 + 32];
    }
    const int jlast_prev = (n - 1 - s) / SB;  // last position of sweep s-1: s + j SB < n
    for (int j = jst;; ++j) {
      const int q0 = s + 1 + j * SB;
      if (q0 >= hi) break;
      const long long t0 = PROF ? clock64() : 0;
      if (s > 0) {
        // (s-1, jd) ran in this range (CTA scope) or in the next one (cluster scope)
        const int jd = min(j + 1, jlast_prev);
        wait_for(s - 1, jd + 1, s + jd * SB >= hi);
      }
      const long long t1 = PROF ? clock64() : 0;
      pw += t1 - t0;
      const int m = min(SB, n - q0);
      double v, tau;
      double* b1 = q0 < lsm ? rowp_g(q0, g, rows) : rowp_g(q0, g, rows);
      const int e1 = q0 < lsm ? lsm : hi;  // end of the first run
      long long* php = ph;
      if (q0 + m <= e1) {
        if (m == SB) s2_task_fast<false, false, PROF>(b1, b1, m, m, j, lane, vp, taup, vs, ws, zs, v, tau, php);
        else s2_task_fast<false, true, PROF>(b1, b1, m, m, j, lane, vp, taup, vs, ws, zs, v, tau, php);
      } else {
        // second run: this range's spill rows, or the next range's first rows (shared memory)
        double* b2 = e1 < hi ? rowp_g(e1, g, rows) : rowp_g(hi, g + 1, rows_nx);
        if (m == SB) s2_task_fast<true, false, PROF>(b1, b2, e1 - q0, m, j, lane, vp, taup, vs, ws, zs, v, tau, php);
        else s2_task_fast<true, true, PROF>(b1, b2, e1 - q0, m, j, lane, vp, taup, vs, ws, zs, v, tau, php);
      }
      // hand-off to the next range, then publish progress
      const int q0n = q0 + SB;
      if (q0n < n && q0n >= hi) {
        hbox_nx[(s % S2_NS) * 33 + lane] = v;
        if (lane == 0) hbox_nx[(s % S2_NS) * 33 + 32] = tau;
      }
      __syncwarp();
      if (lane == 0) {
        // local consumers: (s, j+1) and (s+1, j-1) in this range; the previous range
        // waits only on this sweep's first task here, the next range on the last
        const unsigned t = tag(s, j + 1);
        red_max_rel_cta(my_lp + (s % S2_NS), t);
        if (lp_nx && q0n < n && q0n >= hi) red_max_rel_cl(lp_nx + (s % S2_NS), t);
        if (lp_pv && j == jst) red_max_rel_cl(lp_pv + (s % S2_NS), t);
      }
      vp = v;
      taup = tau;
      if constexpr (PROF) pt += clock64() - t1;
      ++pn;
    }
  }
  if (PROF && lane == 0) {
    long long* q = a.prof + 8 * (blockIdx.x * S2_W + warp);
    q[0] = pw; q[1] = pt; q[2] = pn;
    for (int t = 0; t < 5; ++t) q[3 + t] = ph[t];
  }
  if constexpr (CS > 1) cl.sync(); else __syncthreads();
  for (int s2 = 0; s2 < RPC; ++s2) {
    const int g2 = s2 == 0 ? cr : 2 * CS - 1 - cr;
    const int glo = g2 * R, ghi = min(n, glo + R);
    for (int r = glo + tid; r < ghi; r += S2_W * 32) {
      const double* rr = rowp_g(r, g2, rows);
      a.d[r] = rr[0];
      if (r >= 1) a.e[r - 1] = rr[1];
    }
  }
  if constexpr (CS > 1) cl.sync();
}

template <typename K>
void launch_cluster(Ctx& c, K kern, int cs, dim3 grid, int threads, size_t smem, void** args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(threads);
  lc.dynamicSmemBytes = smem;
  lc.stream = c.stream;
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = cs;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  lc.attrs = &at;
  lc.numAttrs = 1;
  TMB_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
}

void allow_cluster16(Ctx& c, const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({c.device, fn})) return;
  TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done.insert({c.device, fn});
}

template <int CS>
void panel_qr_cs(Ctx& c, const PanelArgs& pa) {
  if (CS > 8) allow_cluster16(c, (const void*)k_panel_qr<CS>);
  PanelArgs a = pa;
  void* args[] = {&a};
  launch_cluster(c, k_panel_qr<CS>, CS, dim3(CS), PQ_NT, 0, args);
  LAUNCHED("k_panel_qr");
}


// ------------------------------------------------------------------ band inverse iteration
// Eigenvectors of the band matrix B for the eigenvalues found on T: for each
// lambda (one warp) the banded LU with partial pivoting of B - lambda I (U has
// 2b superdiagonals; the (b+1) x (2b+1) active window lives in shared memory as
// a circular buffer over rows and columns), then two solves (forward with the
// stored multipliers and row interchanges, back substitution with the stored U)
// from a fixed pseudo-random start (LAPACK dstein's inverse iteration, with a
// zero pivot replaced by eps ||B|| as in dlagtf). Each solve multiplies the
// wanted component by 1 / |lambda - lambda_hat| ~ 1 / (eps ||B||), so the
// result is accurate to eps ||B|| / gap, the class of the twisted factorisation
// it replaces; orthogonality within tight clusters is restored afterwards
// (Newton-Schulz, or the one-stage path when that cannot converge).
constexpr int IV_W = 4;                 // warps (eigenvalues) per block
constexpr int IV_R = SB + 1;            // window rows
constexpr int IV_C = 2 * SB + 1;        // window columns = U row length
constexpr int IV_WIN = (IV_R * IV_C + 1) / 2 * 2;  // window, rounded to 16 bytes
constexpr int IV_SMEM_WARP = (IV_WIN + IV_R + IV_C + 1) / 2 * 2;  // per-warp base stays 16-byte aligned

__device__ __forceinline__ double start_entry(int64_t vi, int64_t i) {
  uint64_t h = (uint64_t)vi * 0x9E3779B97F4A7C15ull ^ ((uint64_t)i + 0x632BE59BD9B4E019ull);
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;  // uniform in [-1, 1)
}

// Gershgorin bound max_r sum_c |B[r][c]| (one block; zero pivots become eps times it)
__global__ void __launch_bounds__(1024) k_band_norm(const double* __restrict__ band, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double mx = 0.0;
  for (int r = threadIdx.x; r < n; r += 1024) {
    double s = 0.0;
    for (int o = 0; o < 2 * SB + 1; ++o) s += fabs(band[(size_t)r * (2 * SB + 1) + o]);
    mx = fmax(mx, s);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (threadIdx.x == 0) *out = mx;
  }
}

__global__ void __launch_bounds__(IV_W * 32) k_band_invit(const double* __restrict__ band, int n, int k,
                                                          const double* __restrict__ vals,
                                                          const double* __restrict__ bnorm,
                                                          double* __restrict__ ub, double* __restrict__ lb,
                                                          int* __restrict__ pb, double* __restrict__ yb,
                                                          double* __restrict__ z) {
  extern __shared__ __align__(16) double smi[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t vi = (int64_t)blockIdx.x * IV_W + warp;
  if (vi >= k) return;
  double* W = smi + (size_t)warp * IV_SMEM_WARP;  // [row % IV_R][col % IV_C]
  double* yw = W + IV_WIN;                        // forward window (IV_R)
  double* xw = yw + IV_R;                         // back window (IV_C)
  const double sigma = vals[vi];
  const double tiny = DBL_EPSILON * fmax(*bnorm, DBL_MIN);
  double* U = ub + (size_t)vi * n * IV_C;
  double* L = lb + (size_t)vi * n * SB;
  int* piv = pb + (size_t)vi * n;
  double* y = yb + (size_t)vi * n;
  double* x = z + (size_t)vi * n;
  auto braw = [&](int r, int cc) -> double {  // B[r][cc], zero outside the band / matrix
    if (r >= n || cc < 0 || cc >= n || cc - r > SB || r - cc > SB) return 0.0;
    return __ldg(band + (size_t)r * IV_C + (cc - r + SB));
  };
  auto bval = [&](int r, int cc) -> double {  // (B - sigma I)[r][cc]
    const double v = braw(r, cc);
    return cc == r && r < n ? v - sigma : v;
  };
  for (int rr = 0; rr < IV_R; ++rr)
    for (int cc = lane; cc < IV_C; cc += 32) W[rr * IV_C + cc] = bval(rr, cc);
  __syncwarp();
  // ---- LU with partial pivoting; the row entering the window (i + b + 1 at
  // the end of step i) is loaded two steps ahead into registers
  double nr[2][3];
  // raw band values (the shift is applied when the row enters the window, so
  // no arithmetic waits on these loads in the step that issues them)
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int off = lane + 32 * u;
      nr[q][u] = (u < 2 || lane == 0) ? braw(IV_R + q, q + 1 + off) : 0.0;
    }
  for (int i = 0; i < n; ++i) {
    const int nw = min(IV_R, n - i);
    const int ci = i % IV_C;
    double cand = -1.0;
    int cr = i;
    if (lane < nw) { cand = fabs(W[((i + lane) % IV_R) * IV_C + ci]); cr = i + lane; }
    if (lane == 0 && nw == IV_R) {
      const double c2 = fabs(W[((i + 32) % IV_R) * IV_C + ci]);
      if (c2 > cand) { cand = c2; cr = i + 32; }
    }
    // row entering after step i + 2
    double nn[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int off = lane + 32 * u;
      nn[u] = (u < 2 || lane == 0) ? braw(i + IV_R + 2, i + 3 + off) : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_xor_sync(FULL, cand, o);
      const int orr = __shfl_xor_sync(FULL, cr, o);
      if (oc > cand || (oc == cand && orr < cr)) { cand = oc; cr = orr; }
    }
    const int pr = cr;
    if (pr != i) {
      double* a0 = W + (i % IV_R) * IV_C;
      double* a1 = W + (pr % IV_R) * IV_C;
      for (int cc = lane; cc < IV_C; cc += 32) { const double t = a0[cc]; a0[cc] = a1[cc]; a1[cc] = t; }
    }
    __syncwarp();
    double* prow = W + (i % IV_R) * IV_C;
    double pv = prow[ci];
    if (pv == 0.0) pv = tiny;
    double ml = 0.0;
    if (lane < nw - 1) ml = W[((i + 1 + lane) % IV_R) * IV_C + ci] / pv;
    L[(size_t)i * SB + lane] = ml;
    if (lane == 0) piv[i] = pr;
    __syncwarp();
    // Row-wise elimination: lane l owns window row i+1+l and updates all its 65
    // column slots against the pivot row at static offsets (column c sits in
    // slot c mod 65, the same in every row), in chunks whose loads all precede
    // their stores (the compiler cannot hoist loads past possibly aliasing
    // stores). Slot i (column i + 65 from now on) is then zeroed.
    if (lane < nw - 1) {
      double* wr = W + ((i + 1 + lane) % IV_R) * IV_C;
      constexpr int CH = 22;
#pragma unroll
      for (int c0 = 0; c0 < IV_C; c0 += CH) {
        double ow[CH], pw[CH];
#pragma unroll
        for (int t = 0; t < CH; ++t)
          if (c0 + t < IV_C) { ow[t] = wr[c0 + t]; pw[t] = prow[c0 + t]; }
#pragma unroll
        for (int t = 0; t < CH; ++t)
          if (c0 + t < IV_C) wr[c0 + t] = fma(-ml, pw[t], ow[t]);
      }
      wr[ci] = 0.0;
    }
    for (int off = lane; off < IV_C; off += 32) {
      const int cc = i + off;
      U[(size_t)i * IV_C + off] = off == 0 ? pv : (cc < n ? prow[cc % IV_C] : 0.0);
    }
    __syncwarp();
    // the next row (i + b + 1) takes row i's slot; column i + 2b + 1 takes column i's
    const int rn = i + IV_R;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int off = lane + 32 * u;
      // the entering row i + b + 1 meets the diagonal at offset 32 (lane 0, u = 1)
      if (u < 2 || lane == 0)
        prow[(i + 1 + off) % IV_C] = (u == 1 && lane == 0 && rn < n) ? nr[0][u] - sigma : nr[0][u];
      nr[0][u] = nr[1][u];
      nr[1][u] = nn[u];
    }
    __syncwarp();
  }
  // ---- two solves: x <- U^-1 L^-1 P y, y = start, then y = x / |x|.
  // Multipliers, pivots and U rows are read PD steps ahead (register ring,
  // the loop unrolled by PD) so the recurrences wait on shared memory only.
  constexpr int PD = 8;
  double scale = 1.0;
  for (int it = 0; it < 2; ++it) {
    auto yin = [&](int r) -> double { return r < n ? (it == 0 ? start_entry(vi, r) : x[r] * scale) : 0.0; };
    for (int rr = lane; rr < IV_R; rr += 32) yw[rr] = yin(rr);
    if (lane == 0) yw[32] = yin(32);
    __syncwarp();
    double lc[PD], yc[PD];
    int pc[PD];
#pragma unroll
    for (int u = 0; u < PD; ++u) {
      lc[u] = u < n ? L[(size_t)u * SB + lane] : 0.0;
      pc[u] = u < n ? piv[u] : u;
      yc[u] = lane == 0 ? yin(u + IV_R) : 0.0;
    }
    for (int i0 = 0; i0 < n; i0 += PD) {
      double ln[PD], yn[PD];
      int pn[PD];
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        const int ii = i0 + PD + u;
        ln[u] = ii < n ? L[(size_t)ii * SB + lane] : 0.0;
        pn[u] = ii < n ? piv[ii] : ii;
        yn[u] = lane == 0 ? yin(ii + IV_R) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        const int i = i0 + u;
        if (i < n) {
          const int pr = pc[u];
          double yi = yw[i % IV_R];
          if (pr != i) {
            const double yp = yw[pr % IV_R];
            __syncwarp();
            if (lane == 0) yw[pr % IV_R] = yi;
            yi = yp;
          }
          __syncwarp();
          if (lane < min(IV_R, n - i) - 1) yw[(i + 1 + lane) % IV_R] = fma(-lc[u], yi, yw[(i + 1 + lane) % IV_R]);
          if (lane == 0) { y[i] = yi; yw[i % IV_R] = yc[u]; }
          __syncwarp();
        }
      }
#pragma unroll
      for (int u = 0; u < PD; ++u) { lc[u] = ln[u]; pc[u] = pn[u]; yc[u] = yn[u]; }
    }
    __syncwarp();
    // back substitution, window x[i+1 .. i+2b]
    for (int cc = lane; cc < IV_C; cc += 32) xw[cc] = 0.0;
    __syncwarp();
    double ss = 0.0;
    double u0c[PD], u1c[PD], rc[PD], ycb[PD];
    auto uld = [&](int i, double& a0, double& a1, double& dg, double& yv) {
      if (i >= 0) {
        const double* ur = U + (size_t)i * IV_C;
        a0 = ur[1 + lane];
        a1 = ur[33 + lane];
        dg = ur[0];
        yv = y[i];
      } else {
        a0 = a1 = 0.0; dg = 1.0; yv = 0.0;
      }
    };
    // y[] was written by lane 0 during the forward pass: make it visible to the warp
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PD; ++u) uld(n - 1 - u, u0c[u], u1c[u], rc[u], ycb[u]);
    for (int i0 = n - 1; i0 >= 0; i0 -= PD) {
      double u0n[PD], u1n[PD], rn[PD], ynb[PD];
#pragma unroll
      for (int u = 0; u < PD; ++u) rc[u] = 1.0 / rc[u];  // this chunk's pivots arrived a chunk ago
#pragma unroll
      for (int u = 0; u < PD; ++u) uld(i0 - PD - u, u0n[u], u1n[u], rn[u], ynb[u]);
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        const int i = i0 - u;
        if (i >= 0) {
          double part = u0c[u] * xw[(i + 1 + lane) % IV_C];
          part = fma(u1c[u], xw[(i + 33 + lane) % IV_C], part);
          part = wsum(part);
          const double xi = (ycb[u] - part) * rc[u];
          __syncwarp();
          if (lane == 0) { xw[i % IV_C] = xi; x[i] = xi; }
          ss = fma(xi, xi, ss);
          __syncwarp();
        }
      }
#pragma unroll
      for (int u = 0; u < PD; ++u) { u0c[u] = u0n[u]; u1c[u] = u1n[u]; rc[u] = rn[u]; ycb[u] = ynb[u]; }
    }
    __syncwarp();
    scale = 1.0 / sqrt(ss);
  }
  for (int i = lane; i < n; i += 32) x[i] *= scale;
}

}  // namespace

// Panels are processed in groups of G with the trailing update deferred to the
// end of the group (one DMMA GEMM with K = 64 G instead of G GEMMs with K = 64,
// which were bound by the C-tile traffic at K = 64). Inside a group, panel q
// first brings its own columns (and diagonal block) up to date, and its X uses
// the stale trailing matrix plus the pending terms (dlatrd's device, restated):
//   X = (A - sum_{q'<q} V_q' W_q'^T + W_q' V_q'^T) VT = A VT - [V W]_{q'} ([W V]_{q'}^T VT).
// The pending [V_q W_q V_q] triples live side by side in VWg (rows from the
// group's first reflector row rg, zero above each panel's own rows).
void sy2sb(Ctx& c, double* A, int64_t n, double* hv, double* tau) {
  static const int genv = [] {
    const char* e = std::getenv("TMB_SBR_GROUP");  // A/B: panels per deferred trailing update
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int G = genv ? genv : (n > 3000 ? 4 : 2);
  const size_t mk = c.arena.mark();
  const int64_t mmax = n - SB;
  double* S = alloc<double>(c, SB * SB);
  double* T = alloc<double>(c, SB * SB);
  double* M = alloc<double>(c, SB * SB);
  double* VT = alloc<double>(c, (size_t)mmax * SB);
  double* X = alloc<double>(c, (size_t)mmax * SB);
  double* Yc = alloc<double>(c, (size_t)G * 2 * SB * SB);
  double* VWg = alloc<double>(c, (size_t)mmax * 3 * SB * G);
  for (int64_t g0 = 0; g0 + SB < n - 1; g0 += (int64_t)G * SB) {
    const int64_t rg = g0 + SB, ldw = n - rg;
    TMB_CUDA(cudaMemsetAsync(VWg, 0, sizeof(double) * ldw * 3 * SB * G, c.stream));
    int q = 0;
    for (; q < G; ++q) {
      const int64_t p0 = g0 + q * SB, r0 = p0 + SB;
      if (!(p0 + SB < n - 1)) break;
      const int64_t m = n - r0;
      if (q > 0) {  // A[p0:, p0:p0+32] -= sum_{q'<q} [V W] [W V]^T (rows p0.., columns of this panel)
        GemmDesc g;
        g.M = n - p0; g.N = SB; g.K1 = 2 * SB; g.K2 = q;
        g.A = VWg + (p0 - rg); g.sAm = 1; g.sAk1 = ldw; g.sAk2 = 3 * SB * ldw;
        g.B = VWg + (p0 - rg) + SB * ldw; g.sBn = 1; g.sBk1 = ldw; g.sBk2 = 3 * SB * ldw;
        g.C = A + p0 + n * p0; g.sCm = 1; g.sCn = n;
        g.alpha = -1.0; g.beta = 1.0;
        gemm(c, g);
      }
      PanelArgs pa{A, n, p0, hv, tau};
      if (m <= PQ_NT) panel_qr_cs<1>(c, pa);
      else if (m <= 2 * PQ_NT) panel_qr_cs<2>(c, pa);
      else if (m <= 4 * PQ_NT) panel_qr_cs<4>(c, pa);
      else if (m <= 8 * PQ_NT) panel_qr_cs<8>(c, pa);
      else if (m <= 16 * PQ_NT) panel_qr_cs<16>(c, pa);
      else throw Error(TMB_EINVAL, "sy2sb: matrix too large for the cluster panel factorisation");
      const double* V = hv + r0 + n * p0;  // m x 32, ld n
      {  // S = V^T V
        GemmDesc g;
        g.M = SB; g.N = SB; g.K1 = m;
        g.A = V; g.sAm = n; g.sAk1 = 1;
        g.B = V; g.sBk1 = 1; g.sBn = n;
        g.C = S; g.sCm = 1; g.sCn = SB;
        gemm(c, g);
      }
      k_larft32<<<1, SB, 0, c.stream>>>(S, tau + p0, T);
      LAUNCHED("k_larft32");
      {  // VT = V T
        GemmDesc g;
        g.M = m; g.N = SB; g.K1 = SB;
        g.A = V; g.sAm = 1; g.sAk1 = n;
        g.B = T; g.sBk1 = 1; g.sBn = SB;
        g.C = VT; g.sCm = 1; g.sCn = m;
        gemm(c, g);
      }
      {  // X = A22 VT (A22 stale by the group's pending updates)
        GemmDesc g;
        g.M = m; g.N = SB; g.K1 = m;
        g.A = A + r0 + n * r0; g.sAm = 1; g.sAk1 = n;
        g.B = VT; g.sBk1 = 1; g.sBn = m;
        g.C = X; g.sCm = 1; g.sCn = m;
        gemm(c, g);
      }
      if (q > 0) {
        GemmDesc y;  // Yc[q'] = [W V]_{q', rows r0..}^T VT  (64 x 32 per pending panel)
        y.M = 2 * SB; y.N = SB; y.K1 = m; y.batch = q;
        y.A = VWg + (r0 - rg) + SB * ldw; y.sAm = ldw; y.sAk1 = 1; y.sAb = 3 * SB * ldw;
        y.B = VT; y.sBk1 = 1; y.sBn = m; y.sBb = 0;
        y.C = Yc; y.sCm = 1; y.sCn = 2 * SB; y.sCb = 2 * SB * SB;
        gemm(c, y);
        GemmDesc x2;  // X -= [V W]_{q', rows r0..} Yc[q']
        x2.M = m; x2.N = SB; x2.K1 = 2 * SB; x2.K2 = q;
        x2.A = VWg + (r0 - rg); x2.sAm = 1; x2.sAk1 = ldw; x2.sAk2 = 3 * SB * ldw;
        x2.B = Yc; x2.sBk1 = 1; x2.sBk2 = 2 * SB * SB; x2.sBn = 2 * SB;
        x2.C = X; x2.sCm = 1; x2.sCn = m;
        x2.alpha = -1.0; x2.beta = 1.0;
        gemm(c, x2);
      }
      {  // M = V^T X
        GemmDesc g;
        g.M = SB; g.N = SB; g.K1 = m;
        g.A = V; g.sAm = n; g.sAk1 = 1;
        g.B = X; g.sBk1 = 1; g.sBn = m;
        g.C = M; g.sCm = 1; g.sCn = SB;
        gemm(c, g);
      }
      k_sbr_w<<<(unsigned)std::min<int64_t>(ceil_div(m, 8), 4 * c.num_sms), 256, 0, c.stream>>>(
          X, V, n, M, T, m, VWg + (r0 - rg) + (int64_t)3 * SB * q * ldw, ldw);
      LAUNCHED("k_sbr_w");
    }
    // the group's deferred two-sided update of everything right of / below its panels
    const int64_t pn = g0 + (int64_t)q * SB;
    if (q > 0 && pn < n) {
      GemmDesc u;
      u.M = n - pn; u.N = n - pn; u.K1 = 2 * SB; u.K2 = q;
      u.A = VWg + (pn - rg); u.sAm = 1; u.sAk1 = ldw; u.sAk2 = 3 * SB * ldw;
      u.B = VWg + (pn - rg) + SB * ldw; u.sBn = 1; u.sBk1 = ldw; u.sBk2 = 3 * SB * ldw;
      u.C = A + pn + n * pn; u.sCm = 1; u.sCn = n;
      u.alpha = -1.0; u.beta = 1.0;
      gemm(c, u);
    }
  }
  c.arena.release(mk);
}

void band_rows(Ctx& c, const double* A, int64_t n, double* band) {
  const int64_t total = n * (2 * SB + 1);
  k_band_rows<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 8 * c.num_sms), 256, 0, c.stream>>>(A, n, band);
  LAUNCHED("k_band_rows");
}

namespace {
template <int RPC>
constexpr size_t s2_fixed() {
  return sizeof(double) * (RPC * S2_NS * 33 + S2_W * 96) + sizeof(unsigned) * RPC * S2_NS;
}
constexpr int S2_MAXRS = (int)((227 * 1024 - s2_fixed<2>()) / (sizeof(double) * S2_LDL));

template <int CS, int RPC>
void sb2st_cs(Ctx& c, const double* band, int n, double* d, double* e) {
  const int R = (n + CS * RPC - 1) / (CS * RPC);  // rows per range
  // rows kept in shared memory per CTA (its RPC ranges back to back); a spill region,
  // when needed, holds >= SB rows so a task's 32 rows never span more than two runs,
  // and every range's first SB rows stay in shared memory
  const int RS = RPC * R <= S2_MAXRS ? RPC * R : std::min(S2_MAXRS, RPC * R - SB);
  if (RPC == 2 && RS < R + SB) throw Error(TMB_EINVAL, "sb2st: band rows do not fit the cluster");
  const size_t smem = s2_fixed<RPC>() + sizeof(double) * (size_t)RS * S2_LDL;
  const size_t mk = c.arena.mark();
  double* spill = RPC * R > RS ? alloc<double>(c, (size_t)CS * (RPC * R - RS) * S2_LDL) : nullptr;
  static const bool prof_on = std::getenv("TMB_S2_PROF") != nullptr;
  const void* kfn = prof_on ? (const void*)k_sb2st<CS, RPC, true> : (const void*)k_sb2st<CS, RPC, false>;
  set_smem_attr(c, kfn, smem);
  if (CS > 8) allow_cluster16(c, kfn);
  long long* prof = nullptr;
  if (prof_on) {
    prof = alloc<long long>(c, (size_t)CS * S2_W * 8);
    TMB_CUDA(cudaMemsetAsync(prof, 0, sizeof(long long) * CS * S2_W * 8, c.stream));
  }
  S2Args a{band, n, R, RS, spill, d, e, prof};
  void* args[] = {&a};
  if (prof_on) launch_cluster(c, k_sb2st<CS, RPC, true>, CS, dim3(CS), S2_W * 32, smem, args);
  else launch_cluster(c, k_sb2st<CS, RPC, false>, CS, dim3(CS), S2_W * 32, smem, args);
  LAUNCHED("k_sb2st");
  if (prof) {
    std::vector<long long> h((size_t)CS * S2_W * 8);
    TMB_CUDA(cudaMemcpyAsync(h.data(), prof, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    for (int b = 0; b < CS; ++b) {
      long long w = 0, t = 0, k = 0, f[5] = {0, 0, 0, 0, 0};
      for (int q = 0; q < S2_W; ++q) {
        const long long* r = &h[(b * S2_W + q) * 8];
        w += r[0]; t += r[1]; k += r[2];
        for (int u = 0; u < 5; ++u) f[u] += r[3 + u];
      }
      const double fk = f[4] ? (double)f[4] : 1.0;
      std::fprintf(stderr, "sb2st n=%d CTA %d: tasks %lld, cycles/task %.0f, wait cycles/task %.0f | fast tasks %lld: "
                   "right %.0f house %.0f left %.0f diag %.0f\n", n, b, k, k ? (double)t / k : 0.0,
                   k ? (double)w / k : 0.0, f[4], f[0] / fk, f[1] / fk, f[2] / fk, f[3] / fk);
    }
  }
  c.arena.release(mk);
}
}  // namespace

void sb2st(Ctx& c, const double* band, int64_t n, double* d, double* e) {
  // rows per range R: >= SB (a task spans at most two ranges) and < 63 x (warps per
  // range) (the warps of one range can never wait on a later sweep they own
  // themselves). TMB_S2_MIRROR=1 pairs mirrored ranges on the 16-CTA cluster (balances
  // the per-CTA task counts; measured slower: n = 7680 244 vs 239 ms, n = 4700 108 vs
  // 105 ms -- half the warps per range, twice the range boundaries)
  static const bool mirror = [] {
    const char* s = std::getenv("TMB_S2_MIRROR");
    return s && std::atoi(s) == 1;
  }();
  const int N = (int)n;
  if (n <= S2_MAXRS) sb2st_cs<1, 1>(c, band, N, d, e);
  else if (n <= 2 * S2_MAXRS) sb2st_cs<2, 1>(c, band, N, d, e);
  else if (n <= 4 * S2_MAXRS) sb2st_cs<4, 1>(c, band, N, d, e);
  else if (n <= 8 * S2_MAXRS) sb2st_cs<8, 1>(c, band, N, d, e);
  else if (mirror && ceil_div(n, 32) < 63 * (S2_W / 2)) sb2st_cs<16, 2>(c, band, N, d, e);
  else if (ceil_div(n, 16) < 63 * S2_W) sb2st_cs<16, 1>(c, band, N, d, e);
  else throw Error(TMB_EINVAL, "sb2st: band too large for one cluster");
}

void band_invit(Ctx& c, const double* band, int64_t n, int64_t k, const double* vals, double* z) {
  const size_t mk = c.arena.mark();
  double* bnorm = alloc<double>(c, 1);
  k_band_norm<<<1, 1024, 0, c.stream>>>(band, (int)n, bnorm);
  LAUNCHED("k_band_norm");
  double* ub = alloc<double>(c, (size_t)k * n * IV_C);
  double* lb = alloc<double>(c, (size_t)k * n * SB);
  int* pb = alloc<int>(c, (size_t)k * n);
  double* yb = alloc<double>(c, (size_t)k * n);
  const size_t smem = sizeof(double) * IV_W * IV_SMEM_WARP;
  set_smem_attr(c, (const void*)k_band_invit, smem);
  k_band_invit<<<(unsigned)ceil_div(k, IV_W), IV_W * 32, smem, c.stream>>>(band, (int)n, (int)k, vals, bnorm, ub,
                                                                           lb, pb, yb, z);
  LAUNCHED("k_band_invit");
  c.arena.release(mk);
}

}  // namespace tmb
