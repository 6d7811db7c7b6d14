// Host-side Tucker-ALS orchestration over the device kernels (tucker.py).
// Native C++ runtime: workspace arena, contraction schedule, sweep loop,
// convergence / best-of bookkeeping. No arithmetic on the host except the
// control-flow scalars (fit, factor change) read back once per sweep.
#include "solver.h"

#include <cstdlib>

namespace tmb {

// ------------------------------------------------------------------ Arena
// Stack-disciplined bump allocator over retained cudaMalloc chunks.
// mark() encodes (chunk index, offset); release() pops back to it.
Arena::~Arena() { free_all(); }

size_t Arena::capacity() const {
  size_t s = 0;
  for (const auto& c : chunks_) s += c.cap;
  return s;
}

void* Arena::alloc(size_t bytes) {
  bytes = std::max<size_t>(256, (bytes + 255) & ~size_t(255));
  const auto track = [&] {
    size_t in_use = 0;
    for (size_t j = 0; j <= cur_ && j < chunks_.size(); ++j) in_use += chunks_[j].used;
    peak_ = std::max(peak_, in_use);
  };
  while (cur_ < chunks_.size()) {
    Chunk& c = chunks_[cur_];
    if (c.cap - c.used >= bytes) {
      void* p = c.p + c.used;
      c.used += bytes;
      track();
      return p;
    }
    if (cur_ + 1 < chunks_.size() && chunks_[cur_ + 1].cap >= bytes) { ++cur_; continue; }
    break;
  }
  const size_t cap = std::max<size_t>(bytes, size_t(64) << 20);
  char* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, cap);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(TMB_ECUDA, "workspace allocation of " + std::to_string(cap) + " bytes failed: " +
                               cudaGetErrorString(e));
  }
  const size_t pos = chunks_.empty() ? 0 : cur_ + 1;
  chunks_.insert(chunks_.begin() + pos, Chunk{p, cap, bytes});
  cur_ = pos;
  track();
  return p;
}

// Called between API calls only (no live allocations; the caller synchronised
// the stream): replaces a smaller pool by one retained chunk of `bytes`.
void Arena::reserve(size_t bytes) {
  if (bytes == 0 || capacity() >= bytes) return;
  free_all();
  alloc(bytes);
  release(0);
}

size_t Arena::mark() const {
  return chunks_.empty() ? 0 : ((cur_ << 40) | chunks_[cur_].used);
}

void Arena::release(size_t m) {
  if (chunks_.empty()) return;
  const size_t idx = m >> 40, used = m & ((size_t(1) << 40) - 1);
  cur_ = std::min(idx, chunks_.size() - 1);
  chunks_[cur_].used = (idx < chunks_.size()) ? used : chunks_[cur_].used;
  for (size_t j = cur_ + 1; j < chunks_.size(); ++j) chunks_[j].used = 0;
}

void Arena::free_all() {
  for (auto& c : chunks_) cudaFree(c.p);
  chunks_.clear();
  cur_ = 0;
}

// ------------------------------------------------------------------ kernel timer
static cudaEvent_t take_event(Ctx& c) {
  KernelTimes& k = c.kt;
  if (k.used == k.pool.size()) {
    cudaEvent_t e;
    TMB_CUDA(cudaEventCreate(&e));
    k.pool.push_back(e);
  }
  return k.pool[k.used++];
}

Timed::Timed(Ctx& c, int tag, double work) : c_(c), tag_(tag), work_(work) {
  if (!c_.timing) return;
  a_ = c_.kt.used;
  TMB_CUDA(cudaEventRecord(take_event(c_), c_.stream));
}

Timed::~Timed() {
  if (!c_.timing) return;
  const size_t b = c_.kt.used;
  if (cudaEventRecord(take_event(c_), c_.stream) == cudaSuccess) c_.kt.recs.push_back({tag_, a_, b, work_});
}

void timing_enable(Ctx& c, bool on) {
  c.timing = on;
  c.kt.used = 0;
  c.kt.recs.clear();
}

void timing_read(Ctx& c, int tag, int64_t* count, double* ms, double* work) {
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  int64_t n = 0;
  double t = 0.0, w = 0.0;
  for (const auto& r : c.kt.recs) {
    if (r.tag != tag) continue;
    float e = 0.f;
    TMB_CUDA(cudaEventElapsedTime(&e, c.kt.pool[r.a], c.kt.pool[r.b]));
    ++n;
    t += e;
    w += r.work;
  }
  *count = n;
  *ms = t;
  *work = w;
}

// ------------------------------------------------------------------ helpers
int64_t prod(const Dims& d, int a, int b) {
  int64_t p = 1;
  for (int i = a; i < b; ++i) p *= d[i];
  return p;
}

// whether ttm_dev sends the (L, K, Rr) -> r contraction to the Ozaki kernel (see ttm_dev)
static bool ozaki_for(int64_t L, int64_t K, int64_t Rr, int64_t r) {
  static const int oz_mode0 = [] {
    const char* e = std::getenv("TMB_OZ_MODE0");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  if (K <= 64 && r <= 64) return false;  // small_ttm
  const double flops = 2.0 * (double)L * Rr * K * r;
  const bool mode0_oz = L == 1 && (oz_mode0 == 1 || (oz_mode0 < 0 && flops >= 2e10));
  return ozaki_enabled() && (L >= 32 || mode0_oz) && flops >= 8e9 && K < 65536 && L * Rr <= 32LL * 65535 - 128;
}

void ttm_dev(Ctx& c, const void* x, DType tx, const Dims& dims, int mode, const double* m, int64_t r,
             int64_t sMr, int64_t sMk, double* y) {
  const int N = (int)dims.size();
  const int64_t L = prod(dims, 0, mode), K = dims[mode], Rr = prod(dims, mode + 1, N);
  if (K <= 64 && r <= 64) {
    small_ttm(c, x, tx, L, K, Rr, m, r, sMr, sMk, y);
    return;
  }
  // full passes over the tensor (>= 8 GFLOP) with the contracted mode not the first:
  // Ozaki int8 digit products on tcgen05 (measured at C2: mode 1 1.62 vs 1.96 ms on
  // DMMA). The mode-0 pass from 20 GFLOP: with the digit planes of the raw tensor kept
  // across the sweeps (ozaki_cache_slot) it saves 9 ms per C2 stack (34 GFLOP passes;
  // 424 -> 415 ms) and 0.24 s per C5 stack (1.9 TFLOP; gemm 1786 -> 1090 ms); C3's
  // 17 GFLOP passes tie. TMB_OZ_MODE0=0 / 1: never / always for mode 0.
  // (launch-grid limit: the digit split and GEMM grids have L*Rr/32 and L*Rr/64 rows in
  // gridDim.y <= 65535; K < 65536 keeps 8*64*64*K digit products inside int32)
  if (ozaki_for(L, K, Rr, r)) {
    ozaki_ttm(c, x, tx, L, K, Rr, m, r, sMr, sMk, y);
    return;
  }
  GemmDesc g;
  if (L == 1) {  // Y(i, rr) = sum_k M(i,k) X(k, rr): one GEMM over the mode-0 unfolding
    g.M = r; g.N = Rr; g.K1 = K;
    g.A = m; g.ta = F64; g.sAm = sMr; g.sAk1 = sMk;
    g.B = x; g.tb = tx; g.sBk1 = 1; g.sBn = K;
    g.C = y; g.sCm = 1; g.sCn = r;
  } else {       // per trailing slab rr: Y_rr(l, i) = sum_k X_rr(l, k) M(i, k)
    g.M = L; g.N = r; g.K1 = K; g.batch = (int)Rr;
    g.A = x; g.ta = tx; g.sAm = 1; g.sAk1 = L; g.sAb = L * K;
    g.B = m; g.tb = F64; g.sBk1 = sMk; g.sBn = sMr;
    g.C = y; g.sCm = 1; g.sCn = L; g.sCb = L * r;
  }
  if (Rr > 32768 && L > 1) {  // grid.z limit: chunk the slabs
    for (int64_t b0 = 0; b0 < Rr; b0 += 32768) {
      GemmDesc h = g;
      h.batch = (int)std::min<int64_t>(32768, Rr - b0);
      h.A = static_cast<const char*>(x) + b0 * L * K * (tx == F32 ? 4 : 8);
      h.C = y + b0 * L * r;
      gemm(c, h);
    }
    return;
  }
  gemm(c, g);
}

void mode_gram_dev(Ctx& c, const void* x, DType tx, const Dims& dims, int mode, double* G) {
  const int N = (int)dims.size();
  const int64_t L = prod(dims, 0, mode), K = dims[mode], Rr = prod(dims, mode + 1, N);
  if (K <= 64) {
    small_gram(c, x, tx, L, K, Rr, G);
    return;
  }
  GemmDesc g;
  g.M = K; g.N = K;
  g.A = x; g.ta = tx; g.B = x; g.tb = tx;
  g.C = G; g.sCm = 1; g.sCn = K;
  g.syrk_upper = true;
  if (L == 1) {  // unfolding is the column-major K x Rr matrix itself
    g.K1 = Rr; g.K2 = 1;
    g.sAm = 1; g.sAk1 = K;
    g.sBn = 1; g.sBk1 = K;
  } else {       // inner index (l, rr): A(i, l, rr) = X[l + L i + L K rr]
    g.K1 = L; g.K2 = Rr;
    g.sAm = L; g.sAk1 = 1; g.sAk2 = L * K;
    g.sBn = L; g.sBk1 = 1; g.sBk2 = L * K;
  }
  gemm(c, g);
  mirror_upper(c, G, K, 1, 0);
}

// Factor as the TTM matrix: transpose -> M = F^T (F is dims[n] x cols, col-major)
static void factor_as_m(const double* f, int64_t frows, int64_t fcols, bool transpose, int64_t* r, int64_t* sMr,
                        int64_t* sMk) {
  if (transpose) { *r = fcols; *sMr = frows; *sMk = 1; }
  else { *r = frows; *sMr = 1; *sMk = frows; }
}

std::vector<int> contraction_order(const Dims& dims, const std::vector<int64_t>& out_rows, int skip, bool greedy) {
  std::vector<int> modes;
  for (int n = 0; n < (int)dims.size(); ++n)
    if (n != skip) modes.push_back(n);
  if (greedy)  // tensor.py:126-135 (stable sort on out_rows / dim)
    std::stable_sort(modes.begin(), modes.end(), [&](int a, int b) {
      return (double)out_rows[a] / (double)dims[a] < (double)out_rows[b] / (double)dims[b];
    });
  return modes;
}

// out = x x_{modes...} factors (ascending or greedy), result written to y.
void ttmc_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const double* const* factors, const int64_t* frows,
              const int64_t* fcols, int skip, bool transpose, bool greedy, double* y) {
  const int N = (int)dims.size();
  std::vector<int64_t> out_rows(N);
  for (int n = 0; n < N; ++n) out_rows[n] = transpose ? fcols[n] : frows[n];
  const std::vector<int> modes = contraction_order(dims, out_rows, skip, greedy);
  if (modes.empty()) {  // nothing to contract: copy
    const int64_t P = prod(dims, 0, N);
    if (tx == F64) copy_d(c, y, static_cast<const double*>(x), P);
    else convert_f32_f64(c, static_cast<const float*>(x), y, P);
    return;
  }
  const size_t mk = c.arena.mark();
  Dims cur = dims;
  const void* src = x;
  DType st = tx;
  for (size_t q = 0; q < modes.size(); ++q) {
    const int n = modes[q];
    int64_t r, sMr, sMk;
    factor_as_m(factors[n], frows[n], fcols[n], transpose, &r, &sMr, &sMk);
    Dims nd = cur;
    nd[n] = r;
    double* dst = (q + 1 == modes.size()) ? y : alloc<double>(c, (size_t)prod(nd, 0, N));
    ttm_dev(c, src, st, cur, n, factors[n], r, sMr, sMk, dst);
    src = dst;
    st = F64;
    cur = nd;
  }
  c.arena.release(mk);
}

// ------------------------------------------------------------------ Tucker steps
void t_hosvd_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks, bool greedy, double* core,
                 double* const* factors) {
  const int N = (int)dims.size();
  const size_t mk = c.arena.mark();
  for (int n = 0; n < N; ++n) {  // tucker.py:141-145
    double* G = alloc<double>(c, (size_t)dims[n] * dims[n]);
    double* vals = alloc<double>(c, (size_t)ranks[n]);
    mode_gram_dev(c, x, tx, dims, n, G);
    leading_eigvecs(c, G, dims[n], ranks[n], factors[n], vals);
    c.arena.release(mk);
  }
  ttmc_dev(c, x, tx, dims, factors, dims.data(), ranks.data(), -1, true, greedy, core);  // tucker.py:146
}

// Gauss-Seidel sweep (tucker.py:151-163). Ascending order uses the memoised
// prefix P_n = t x_0 S_0^T ... x_n S_n^T (updated factors): Y^(n) = P_{n-1}
// x_{n+1} ... x_{N-1}, the same association order as ttmc(skip=n), with 2 full
// passes over t per sweep instead of N+1.
void hooi_sweep_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks,
                    const double* const* fin, bool greedy, double* core, double* const* fout) {
  const int N = (int)dims.size();
  std::vector<const double*> cur(fin, fin + N);
  const size_t mk = c.arena.mark();
  if (greedy) {
    for (int n = 0; n < N; ++n) {
      Dims yd = ranks;
      yd[n] = dims[n];
      double* Y = alloc<double>(c, (size_t)prod(yd, 0, N));
      ttmc_dev(c, x, tx, dims, cur.data(), dims.data(), ranks.data(), n, true, true, Y);
      double* G = alloc<double>(c, (size_t)dims[n] * dims[n]);
      double* vals = alloc<double>(c, (size_t)ranks[n]);
      mode_gram_dev(c, Y, F64, yd, n, G);
      double* nf = (fout[n] == fin[n]) ? alloc<double>(c, (size_t)dims[n] * ranks[n]) : fout[n];
      leading_eigvecs(c, G, dims[n], ranks[n], nf, vals);
      if (nf != fout[n]) copy_d(c, fout[n], nf, dims[n] * ranks[n]);
      cur[n] = fout[n];
    }
    ttmc_dev(c, x, tx, dims, cur.data(), dims.data(), ranks.data(), -1, true, true, core);
    c.arena.release(mk);
    return;
  }
  static const bool fuse_off = std::getenv("TMB_NO_TTM2") != nullptr;  // A/B: separate small-mode passes
  const void* P = x;  // prefix product with updated factors 0..n-1
  DType pt = tx;
  Dims pd = dims;
  for (int n = 0; n < N; ++n) {
    // Y^(n) = P x_{n+1} S_{n+1}^T ... x_{N-1} S_{N-1}^T
    const void* Y = P;
    DType yt = pt;
    Dims yd = pd;
    for (int m = n + 1; m < N; ++m) {
      Dims nd = yd;
      nd[m] = ranks[m];
      // two trailing small modes (colour, view-exposure): one fused pass
      if (m + 1 < N && !fuse_off && yd[m] <= 64 && ranks[m] <= 64 && yd[m + 1] <= 64 && ranks[m + 1] <= 64) {
        Dims nd2 = nd;
        nd2[m + 1] = ranks[m + 1];
        double* dst = alloc<double>(c, (size_t)prod(nd2, 0, N));
        if (small_ttm2(c, Y, yt, prod(yd, 0, m), yd[m], yd[m + 1], prod(yd, m + 2, N), cur[m], ranks[m], dims[m], 1,
                       cur[m + 1], ranks[m + 1], dims[m + 1], 1, dst)) {
          Y = dst; yt = F64; yd = nd2;
          ++m;
          continue;
        }
      }
      double* dst = alloc<double>(c, (size_t)prod(nd, 0, N));
      ttm_dev(c, Y, yt, yd, m, cur[m], ranks[m], dims[m], 1, dst);
      Y = dst; yt = F64; yd = nd;
    }
    double* G = alloc<double>(c, (size_t)dims[n] * dims[n]);
    double* vals = alloc<double>(c, (size_t)ranks[n]);
    mode_gram_dev(c, Y, yt, yd, n, G);
    double* nf = (fout[n] == fin[n]) ? alloc<double>(c, (size_t)dims[n] * ranks[n]) : fout[n];
    leading_eigvecs(c, G, dims[n], ranks[n], nf, vals);
    cur[n] = nf;
    // P <- P x_n S_n^T
    Dims nd = pd;
    nd[n] = ranks[n];
    double* dst = (n + 1 == N) ? core : alloc<double>(c, (size_t)prod(nd, 0, N));
    ttm_dev(c, P, pt, pd, n, nf, ranks[n], dims[n], 1, dst);
    P = dst; pt = F64; pd = nd;
  }
  for (int n = 0; n < N; ++n)
    if (cur[n] != fout[n]) copy_d(c, fout[n], cur[n], dims[n] * ranks[n]);
  c.arena.release(mk);
}

void reconstruct_dev(Ctx& c, const Dims& ranks, const Dims& dims, const double* core, const double* const* factors,
                     double* out) {
  const int N = (int)dims.size();
  std::vector<int64_t> frows(dims.begin(), dims.end()), fcols(ranks.begin(), ranks.end());
  ttmc_dev(c, core, F64, ranks, factors, frows.data(), fcols.data(), -1, false, false, out);  // tucker.py:166-171
  (void)N;
}

// ||t - reconstruct(model)||^2 (tucker.py:166-171, fit(method="residual")
// tucker.py:186-188) with the K9 fused epilogue: modes 0..N-3 as in
// reconstruct_dev (ascending), then the last two small-mode products and the
// residual in one pass, so the full reconstruction is never written.
void reconstruct_resid_dev(Ctx& c, const Dims& ranks, const Dims& dims, const double* core,
                           const double* const* factors, const void* t, DType tt, double* sse_dev) {
  const int N = (int)dims.size();
  const size_t mk = c.arena.mark();
  bool fused = false;
  if (N >= 3) {
    Dims cur = ranks;
    const double* src = core;
    for (int n = 0; n < N - 2; ++n) {
      Dims nd = cur;
      nd[n] = dims[n];
      double* dst = alloc<double>(c, (size_t)prod(nd, 0, N));
      ttm_dev(c, src, F64, cur, n, factors[n], dims[n], 1, dims[n], dst);  // y = x x_n S_n (S_n: dims x ranks)
      src = dst;
      cur = nd;
    }
    const int a = N - 2, b = N - 1;
    fused = small_ttm2_resid(c, src, prod(cur, 0, a), ranks[a], ranks[b], 1, factors[a], dims[a], 1, dims[a],
                             factors[b], dims[b], 1, dims[b], t, tt, sse_dev);
  }
  if (!fused) {
    double* rec = alloc<double>(c, (size_t)prod(dims, 0, N));
    reconstruct_dev(c, ranks, dims, core, factors, rec);
    resid2_async(c, t, tt, rec, prod(dims, 0, N), sse_dev);
  }
  c.arena.release(mk);
}

// ------------------------------------------------------------------ pairwise perturbation
// tucker.py:199-311. Operators persist across sweeps (own cudaMalloc buffers,
// outside the per-sweep arena); rebuilt only when the PP phase refreshes.
// PPOps / DevBuf are declared in solver.h (the C ABI's tmb_pp handle wraps one).

Dims pp_node_dims(const Dims& dims, const Dims& ranks, unsigned free_modes) {
  Dims d(dims.size());
  for (size_t n = 0; n < dims.size(); ++n) d[n] = ((free_modes >> n) & 1u) ? dims[n] : ranks[n];
  return d;
}

// Memoised dimension tree: the parent of a node re-adds its largest contracted
// mode, so every node is an ascending contraction (tucker.py:238-252).
static std::pair<const void*, DType> pp_node(Ctx& c, PPOps& ops, const void* x, DType tx, unsigned free_modes) {
  const Dims& dims = ops.dims;
  const Dims& ranks = ops.ranks;
  const int N = (int)dims.size();
  const unsigned all = (1u << N) - 1u;
  if (free_modes == all) return {x, tx};
  if (const double* got = ops.find(free_modes)) return {got, F64};
  if (!x) throw Error(TMB_EINVAL, "pp operator " + std::to_string(free_modes) + " was not built");
  int m = N - 1;
  while ((free_modes >> m) & 1u) --m;
  const auto parent = pp_node(c, ops, x, tx, free_modes | (1u << m));
  DevBuf out((size_t)prod(pp_node_dims(dims, ranks, free_modes), 0, N));
  ttm_dev(c, parent.first, parent.second, pp_node_dims(dims, ranks, free_modes | (1u << m)), m, ops.anchors[m].p,
          ranks[m], dims[m], 1, out.p);
  ops.count++;
  ops.nodes.emplace_back(free_modes, std::move(out));
  return {ops.nodes.back().second.p, F64};
}

// pp_operators (tucker.py:222-265): every skip-one and skip-two operator
void pp_build(Ctx& c, PPOps& ops, const void* x, DType tx, const Dims& dims, const Dims& ranks,
              const double* const* anchors) {
  const int N = (int)dims.size();
  ops.dims = dims;
  ops.ranks = ranks;
  ops.nodes.clear();
  ops.anchors.clear();
  ops.deltas.clear();
  ops.nonzero.assign(N, 0);
  ops.count = 0;
  for (int n = 0; n < N; ++n) {
    ops.anchors.emplace_back((size_t)dims[n] * ranks[n]);
    copy_d(c, ops.anchors.back().p, anchors[n], dims[n] * ranks[n]);
    ops.deltas.emplace_back((size_t)dims[n] * ranks[n]);
    TMB_CUDA(cudaMemsetAsync(ops.deltas.back().p, 0, sizeof(double) * dims[n] * ranks[n], c.stream));
  }
  for (int n = 0; n < N; ++n) pp_node(c, ops, x, tx, 1u << n);                  // op_single
  for (int i = 0; i < N; ++i)
    for (int n = i + 1; n < N; ++n) pp_node(c, ops, x, tx, (1u << i) | (1u << n));  // op_pair
}

// PPState.set_current (tucker.py:212-213: deltas = factors - anchors) when
// `factors` is true, else the deltas themselves are given (PPState.deltas = ...);
// returns max_rel_delta (tucker.py:215-219) and records which deltas are nonzero.
double pp_set_deltas(Ctx& c, PPOps& ops, const double* const* src, bool factors) {
  const int N = (int)ops.dims.size();
  const size_t mk = c.arena.mark();
  double* sc = alloc<double>(c, 2 * (size_t)N);
  for (int n = 0; n < N; ++n) {
    const int64_t cnt = ops.dims[n] * ops.ranks[n];
    copy_d(c, ops.deltas[n].p, src[n], cnt);
    if (factors) axpy(c, cnt, -1.0, ops.anchors[n].p, ops.deltas[n].p);
    sumsq_async(c, ops.deltas[n].p, F64, cnt, sc + 2 * n);
    sumsq_async(c, ops.anchors[n].p, F64, cnt, sc + 2 * n + 1);
  }
  std::vector<double> h(2 * (size_t)N);
  TMB_CUDA(cudaMemcpyAsync(h.data(), sc, sizeof(double) * 2 * N, cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  c.arena.release(mk);
  double out = 0.0;
  for (int n = 0; n < N; ++n) {
    ops.nonzero[n] = h[2 * n] > 0.0 ? 1 : 0;  // np.any(d) (tucker.py:275)
    out = std::max(out, std::sqrt(h[2 * n]) / std::sqrt(h[2 * n + 1]));
  }
  return out;
}

// pp_sweep (tucker.py:285-311) from the stored entry deltas: operand
// Y_n = op_single[n] + sum_{i != n, d_i != 0} pair(i, n) x_i d_i^T, the
// corrections summed first in ascending i and then added to op_single
// (_pp_operand, tucker.py:268-282, in the reference's order), then the
// leading eigenvectors of its mode-n Gram; core = Y_{N-1} x_{N-1} S_{N-1}^T
// when core_out is given (the pp estimate), operands copied out when given.
void pp_sweep_dev(Ctx& c, PPOps& ops, double* const* fout, double* core_out, double* const* operands_out) {
  const Dims& dims = ops.dims;
  const Dims& ranks = ops.ranks;
  const int N = (int)dims.size();
  const size_t mk = c.arena.mark();
  const double* last_y = nullptr;
  Dims last_d;
  for (int n = 0; n < N; ++n) {
    const Dims yd = pp_node_dims(dims, ranks, 1u << n);
    const int64_t ysz = prod(yd, 0, N);
    const double* single = ops.find(1u << n);
    if (!single) throw Error(TMB_EINVAL, "pp operators not built");
    double* acc = nullptr;
    double* tmp = alloc<double>(c, (size_t)ysz);
    for (int i = 0; i < N; ++i) {
      if (i == n || !ops.nonzero[i]) continue;
      const unsigned pm = (1u << i) | (1u << n);
      const double* pair = ops.find(pm);
      double* dst = acc ? tmp : alloc<double>(c, (size_t)ysz);
      ttm_dev(c, pair, F64, pp_node_dims(dims, ranks, pm), i, ops.deltas[i].p, ranks[i], dims[i], 1, dst);  // x_i d_i^T
      if (acc) axpy(c, ysz, 1.0, tmp, acc);
      else acc = dst;
    }
    const double* y = single;
    if (acc) {
      axpy(c, ysz, 1.0, single, acc);  // y + acc (fp addition is commutative)
      y = acc;
    }
    if (operands_out && operands_out[n]) copy_d(c, operands_out[n], y, ysz);
    double* G = alloc<double>(c, (size_t)dims[n] * dims[n]);
    double* vals = alloc<double>(c, (size_t)ranks[n]);
    mode_gram_dev(c, y, F64, yd, n, G);
    leading_eigvecs(c, G, dims[n], ranks[n], fout[n], vals);
    last_y = y;
    last_d = yd;
  }
  if (core_out) ttm_dev(c, last_y, F64, last_d, N - 1, fout[N - 1], ranks[N - 1], dims[N - 1], 1, core_out);
  c.arena.release(mk);
}

// ------------------------------------------------------------------ driver
static double fit_from(double tn, double core_sumsq) {
  // tucker.py:181-191 with fro_norm = sqrt(sum of squares)
  const double cn = std::sqrt(core_sumsq);
  const double resid = std::sqrt(std::max(tn * tn - cn * cn, 0.0));
  return 1.0 - resid / tn;
}

void tucker_als_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks, const tmb_solve_cfg& cfg,
                    double* core_out, double* const* factors_out, tmb_trace* trace) {
  const int N = (int)dims.size();
  const int64_t P = prod(dims, 0, N), Pc = prod(ranks, 0, N);
  const bool greedy = cfg.sequential_reduction == 0;
  const double tsq = sumsq(c, x, tx, P);
  const double tn = std::sqrt(tsq);
  if (tn == 0.0) throw Error(TMB_EINVAL, "cannot decompose the zero tensor");  // tucker.py:341-342
  const size_t mk = c.arena.mark();
  // the two full passes over the raw tensor every sweep (mode 1, then mode 0 after the
  // mode-0 update) re-split the same operand: keep its Ozaki digit planes for the solve
  // (C2: the 498 MB mode-1 planes; C5: 14.3 GB per pass). Also used by the T-HOSVD core.
  c.oz_clear();
  if (N >= 2) {
    int slot = 0;
    if (ozaki_for(dims[0], dims[1], prod(dims, 2, N), ranks[1]))
      ozaki_cache_slot(c, slot++, x, tx, dims[0], dims[1], prod(dims, 2, N));
    if (ozaki_for(1, dims[0], prod(dims, 1, N), ranks[0]))
      ozaki_cache_slot(c, slot++, x, tx, 1, dims[0], prod(dims, 1, N));
  }
  // model buffers: current (a), candidate (b), best
  auto model_alloc = [&](std::vector<double*>& f) -> double* {
    f.resize(N);
    for (int n = 0; n < N; ++n) f[n] = alloc<double>(c, (size_t)dims[n] * ranks[n]);
    return alloc<double>(c, (size_t)Pc);
  };
  std::vector<double*> fa, fb, fbest;
  double* ca = model_alloc(fa);
  double* cb = model_alloc(fb);
  double* cbest = model_alloc(fbest);
  double* scal = alloc<double>(c, 2 + 2 * N);  // [core sumsq, -, per-mode diff/base pairs]
  auto rec = [&](int kind, double fit, double change) {
    if (!trace) return;
    if (trace->n_records >= trace->capacity) throw Error(TMB_EINVAL, "trace capacity too small");
    trace->kind[trace->n_records] = kind;
    trace->fit[trace->n_records] = fit;
    trace->max_change[trace->n_records] = change;
    trace->n_records++;
  };
  if (trace) { trace->n_records = 0; trace->converged = 0; trace->best_index = 0; }

  t_hosvd_dev(c, x, tx, dims, ranks, greedy, ca, fa.data());  // tucker.py:346
  sumsq_async(c, ca, F64, Pc, scal);
  TMB_CUDA(cudaMemcpyAsync(c.host_pinned, scal, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  double cur_fit = fit_from(tn, c.host_pinned[0]);
  rec(TMB_KIND_INIT, cur_fit, std::nan(""));
  double best_fit = cur_fit;
  int best_idx = 0;
  copy_d(c, cbest, ca, Pc);  // tucker.py:349 best = (fit0, init model)
  for (int n = 0; n < N; ++n) copy_d(c, fbest[n], fa[n], dims[n] * ranks[n]);
  bool converged = false;
  if (cur_fit >= 1.0 - cfg.fit_tol) converged = true;  // tucker.py:351-353
  bool phase_pp = false;
  double* cc = ca;
  std::vector<double*>* fc = &fa;
  double* cn = cb;
  std::vector<double*>* fn = &fb;
  PPOps pp;
  std::vector<int64_t> frows(dims.begin(), dims.end()), fcols(ranks.begin(), ranks.end());
  auto read_scalars = [&](int count) {
    TMB_CUDA(cudaMemcpyAsync(c.host_pinned, scal, sizeof(double) * count, cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
  };
  for (int sweep = 1; !converged && sweep <= cfg.max_sweeps; ++sweep) {
    int kind = TMB_KIND_STANDARD;
    bool have_candidate = false;
    if (phase_pp) {  // tucker.py:359-371
      const double max_rel = pp_set_deltas(c, pp, fc->data(), true);  // set_current + max_rel_delta
      if (max_rel <= cfg.pp_exit_tol) {
        pp_sweep_dev(c, pp, fn->data(), nullptr, nullptr);
        ttmc_dev(c, x, tx, dims, fn->data(), frows.data(), fcols.data(), -1, true, greedy, cn);  // _exact_core
        sumsq_async(c, cn, F64, Pc, scal);
        read_scalars(1);
        have_candidate = !(fit_from(tn, c.host_pinned[0]) < cur_fit - 1e-6);  // PP_DIP_TOL, tucker.py:365-366
      }
      if (have_candidate) {
        kind = TMB_KIND_PP;
      } else {  // drifted or regressed: refresh with a standard sweep and new anchors
        hooi_sweep_dev(c, x, tx, dims, ranks, fc->data(), greedy, cn, fn->data());
        pp_build(c, pp, x, tx, dims, ranks, fn->data());
      }
    } else {
      hooi_sweep_dev(c, x, tx, dims, ranks, fc->data(), greedy, cn, fn->data());  // tucker.py:373
    }
    sumsq_async(c, cn, F64, Pc, scal);
    for (int n = 0; n < N; ++n) diff_norms(c, (*fn)[n], (*fc)[n], dims[n] * ranks[n], scal + 2 + 2 * n);
    TMB_CUDA(cudaMemcpyAsync(c.host_pinned, scal, sizeof(double) * (2 + 2 * N), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    double change = 0.0;  // tucker.py:319-323
    for (int n = 0; n < N; ++n)
      change = std::max(change, std::sqrt(c.host_pinned[2 + 2 * n]) / std::sqrt(c.host_pinned[3 + 2 * n]));
    const double new_fit = fit_from(tn, c.host_pinned[0]);
    rec(kind, new_fit, change);
    if (new_fit > best_fit) {  // tucker.py:382-383 (strict)
      best_fit = new_fit;
      best_idx = sweep;
      copy_d(c, cbest, cn, Pc);
      for (int n = 0; n < N; ++n) copy_d(c, fbest[n], (*fn)[n], dims[n] * ranks[n]);
    }
    if (kind == TMB_KIND_STANDARD && !phase_pp && cfg.pp_enter_tol > 0 && change < cfg.pp_enter_tol) {
      phase_pp = true;  // tucker.py:385-387
      pp_build(c, pp, x, tx, dims, ranks, fn->data());
    }
    const bool done = std::fabs(new_fit - cur_fit) < cfg.fit_tol;            // tucker.py:389
    std::swap(cc, cn);
    std::swap(fc, fn);
    cur_fit = new_fit;
    if (done) converged = true;
  }
  // tucker.py:395-396: best-fit model when not converged
  const double* out_core = cc;
  std::vector<double*>* out_f = fc;
  int out_idx = trace ? trace->n_records - 1 : 0;
  if (!converged) {
    out_idx = best_idx;
    out_core = cbest;
    out_f = &fbest;
  }
  copy_d(c, core_out, out_core, Pc);
  for (int n = 0; n < N; ++n) copy_d(c, factors_out[n], (*out_f)[n], dims[n] * ranks[n]);
  if (trace) { trace->converged = converged ? 1 : 0; trace->best_index = out_idx; }
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  c.oz_clear();
  c.arena.release(mk);
}

}  // namespace tmb
