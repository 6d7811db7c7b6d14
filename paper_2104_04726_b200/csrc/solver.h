// Host-side solver entry points (solver.cu), shared with the C ABI (capi.cu).
#pragma once
#include "tmb_internal.cuh"

namespace tmb {

using Dims = std::vector<int64_t>;

int64_t prod(const Dims& d, int a, int b);
void timing_enable(Ctx& c, bool on);
void timing_read(Ctx& c, int tag, int64_t* count, double* ms, double* work);
void ttm_dev(Ctx& c, const void* x, DType tx, const Dims& dims, int mode, const double* m, int64_t r,
             int64_t sMr, int64_t sMk, double* y);
void mode_gram_dev(Ctx& c, const void* x, DType tx, const Dims& dims, int mode, double* G);
void ttmc_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const double* const* factors, const int64_t* frows,
              const int64_t* fcols, int skip, bool transpose, bool greedy, double* y);
void t_hosvd_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks, bool greedy, double* core,
                 double* const* factors);
void hooi_sweep_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks,
                    const double* const* fin, bool greedy, double* core, double* const* fout);
void reconstruct_dev(Ctx& c, const Dims& ranks, const Dims& dims, const double* core, const double* const* factors,
                     double* out);
void reconstruct_resid_dev(Ctx& c, const Dims& ranks, const Dims& dims, const double* core,
                           const double* const* factors, const void* t, DType tt, double* sse_dev);
// pairwise-perturbation operators (tucker.py:199-311): device buffers that outlive the arena
struct DevBuf {
  double* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t count) { TMB_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double))); }
  ~DevBuf() { if (p) cudaFree(p); }
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { if (p) cudaFree(p); p = o.p; o.p = nullptr; }
    return *this;
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

struct PPOps {
  Dims dims, ranks;
  std::vector<DevBuf> anchors;                     // anchor factors (column-major s_n x r_n)
  std::vector<DevBuf> deltas;                      // entry deltas d_n = f_n - a_n
  std::vector<char> nonzero;                       // np.any(d_n)
  std::vector<std::pair<unsigned, DevBuf>> nodes;  // free-mode bitmask -> operator (F-order)
  int count = 0;                                   // contractions evaluated (13 for N = 4)
  const double* find(unsigned m) const {
    for (const auto& kv : nodes)
      if (kv.first == m) return kv.second.p;
    return nullptr;
  }
};
Dims pp_node_dims(const Dims& dims, const Dims& ranks, unsigned free_modes);
void pp_build(Ctx& c, PPOps& ops, const void* x, DType tx, const Dims& dims, const Dims& ranks,
              const double* const* anchors);
double pp_set_deltas(Ctx& c, PPOps& ops, const double* const* src, bool factors);
void pp_sweep_dev(Ctx& c, PPOps& ops, double* const* fout, double* core_out, double* const* operands_out);

void tucker_als_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks, const tmb_solve_cfg& cfg,
                    double* core_out, double* const* factors_out, tmb_trace* trace);

}  // namespace tmb
