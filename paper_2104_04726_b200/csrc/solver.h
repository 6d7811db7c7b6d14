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
void tucker_als_dev(Ctx& c, const void* x, DType tx, const Dims& dims, const Dims& ranks, const tmb_solve_cfg& cfg,
                    double* core_out, double* const* factors_out, tmb_trace* trace);

}  // namespace tmb
