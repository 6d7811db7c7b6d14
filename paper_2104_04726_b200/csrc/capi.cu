// extern "C" boundary (include/tmb.h). Validation happens here, before any
// launch, with the reference's ValueError wording; every C++ exception is
// turned into a status code plus tmb_last_error() text.
#include <cstring>

#include "solver.h"

struct tmb_ctx {
  tmb::Ctx c;
};

struct tmb_pp {
  tmb::PPOps ops;
  int device = 0;
};

namespace {

using tmb::Dims;
using tmb::Error;

template <typename F>
int guard(tmb_ctx* ctx, F&& f) {
  if (!ctx) return TMB_EINVAL;
  ctx->c.err.clear();
  // workspace mark: a throwing call skips its frames' arena releases, so the
  // guard rewinds the arena to where the call started (after the stream has
  // drained any work that may still use it)
  const size_t mk = ctx->c.arena.mark();
  auto rewind = [&]() {
    cudaStreamSynchronize(ctx->c.stream);
    cudaGetLastError();
    ctx->c.oz_clear();  // cache slots point into the released arena frame
    ctx->c.arena.release(mk);
  };
  try {
    TMB_CUDA(cudaSetDevice(ctx->c.device));
    f(ctx->c);
    return TMB_OK;
  } catch (const Error& e) {
    ctx->c.err = e.what();
    rewind();
    return e.code;
  } catch (const std::exception& e) {
    ctx->c.err = e.what();
    rewind();
    return TMB_ECUDA;
  }
}

Dims to_dims(int order, const int64_t* dims) {
  if (order < 1 || order > 16 || !dims) throw Error(TMB_EINVAL, "tensor order must be in [1, 16]");
  Dims d(dims, dims + order);
  for (auto v : d)
    if (v < 1) throw Error(TMB_EINVAL, "all dimensions must be >= 1");
  return d;
}

tmb::DType to_dtype(int t) {
  if (t != TMB_F32 && t != TMB_F64) throw Error(TMB_EINVAL, "dtype must be TMB_F32 or TMB_F64");
  return t == TMB_F32 ? tmb::F32 : tmb::F64;
}

Dims check_ranks(const Dims& dims, const int64_t* ranks) {
  Dims r(ranks, ranks + dims.size());
  for (size_t n = 0; n < dims.size(); ++n)
    if (r[n] < 1 || r[n] > dims[n])  // tucker.py:89-91
      throw Error(TMB_EINVAL, "mode " + std::to_string(n) + ": rank " + std::to_string(r[n]) + " not in [1, " +
                                  std::to_string(dims[n]) + "]");
  return r;
}

}  // namespace

extern "C" {

int tmb_version(void) { return 1; }

int tmb_ctx_create(int device, void* stream, tmb_ctx** out) {
  if (!out) return TMB_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return TMB_ECUDA;
  }
  if (device < 0 || device >= ndev) return TMB_EINVAL;
  auto* ctx = new tmb_ctx();
  ctx->c.device = device;
  ctx->c.stream = static_cast<cudaStream_t>(stream);
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&ctx->c.num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaMallocHost(&ctx->c.host_pinned, 4096) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return TMB_ECUDA;
  }
  *out = ctx;
  return TMB_OK;
}

int tmb_ctx_destroy(tmb_ctx* ctx) {
  if (!ctx) return TMB_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  ctx->c.arena.free_all();
  if (ctx->c.host_pinned) cudaFreeHost(ctx->c.host_pinned);
  delete ctx;
  return TMB_OK;
}

int tmb_ctx_set_stream(tmb_ctx* ctx, void* stream) {
  if (!ctx) return TMB_EINVAL;
  ctx->c.stream = static_cast<cudaStream_t>(stream);
  return TMB_OK;
}

const char* tmb_last_error(const tmb_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int64_t tmb_launch_count(const tmb_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int tmb_workspace_size(const tmb_ctx* ctx, int64_t* reserved_bytes, int64_t* peak_bytes) {
  if (!ctx) return TMB_EINVAL;
  if (reserved_bytes) *reserved_bytes = (int64_t)ctx->c.arena.capacity();
  if (peak_bytes) *peak_bytes = (int64_t)ctx->c.arena.peak();
  return TMB_OK;
}

int tmb_workspace_reserve(tmb_ctx* ctx, int64_t bytes) {
  if (bytes < 0) return TMB_EINVAL;
  return guard(ctx, [&](tmb::Ctx& c) {
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    c.arena.reserve((size_t)bytes);
  });
}

int tmb_timing(tmb_ctx* ctx, int enable) {
  return guard(ctx, [&](tmb::Ctx& c) { tmb::timing_enable(c, enable != 0); });
}

int tmb_timing_read(tmb_ctx* ctx, int tag, int64_t* count, double* ms, double* work) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (tag < 0 || tag >= tmb::TAG_COUNT) throw Error(TMB_EINVAL, "unknown timer tag");
    tmb::timing_read(c, tag, count, ms, work);
  });
}

int tmb_color_u8(tmb_ctx* ctx, const uint8_t* rgb, int64_t n_img, int64_t h, int64_t w, int space, float* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    if (n_img < 0 || h < 0 || w < 0) throw Error(TMB_EINVAL, "negative image extent");
    tmb::color_u8(c, rgb, n_img, h, w, space, out);
  });
}

int tmb_color_u8_channels(tmb_ctx* ctx, const uint8_t* rgb, int64_t n_img, int64_t h, int64_t w, int space,
                          float* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    if (n_img < 0 || h < 0 || w < 0) throw Error(TMB_EINVAL, "negative image extent");
    tmb::color_u8(c, rgb, n_img, h, w, space, out, true);
  });
}

int tmb_varint_encode(tmb_ctx* ctx, const int64_t* levels, int64_t n, uint8_t* out, int64_t cap, int64_t* nbytes) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (n < 0 || cap < 0) throw Error(TMB_EINVAL, "negative size");
    const int64_t b = tmb::varint_encode(c, levels, n, out, cap);
    if (nbytes) *nbytes = b;
  });
}

int tmb_varint_decode(tmb_ctx* ctx, const uint8_t* in, int64_t nbytes, int64_t count, int64_t* levels,
                      int64_t* used) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (nbytes < 0 || count < 0) throw Error(TMB_EINVAL, "negative size");
    const int64_t u = tmb::varint_decode(c, in, nbytes, count, levels);
    if (used) *used = u;
  });
}

int tmb_color_f64(tmb_ctx* ctx, const double* px, int64_t npx, int space, double* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    tmb::color_f64(c, px, npx, space, out);
  });
}

int tmb_color_inv_f64(tmb_ctx* ctx, const double* px, int64_t npx, int space, double* out, int64_t* ncl) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    tmb::color_inv_f64(c, px, npx, space, out, ncl);
  });
}

int tmb_decode_sse(tmb_ctx* ctx, const double* tensor, int64_t n_img, int64_t h, int64_t w, int space,
                   const uint8_t* rgb, double* out_rgb, double* sse_host) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    if (n_img < 0 || h < 0 || w < 0) throw Error(TMB_EINVAL, "negative stack shape");
    if (rgb && !sse_host) throw Error(TMB_EINVAL, "sse_host is required with reference images");
    const size_t mk = c.arena.mark();
    double* sse = rgb ? tmb::alloc<double>(c, (size_t)std::max<int64_t>(n_img, 1)) : nullptr;
    tmb::decode_sse(c, tensor, n_img, h, w, space, rgb, out_rgb, sse);
    if (rgb && n_img > 0) {
      TMB_CUDA(cudaMemcpyAsync(sse_host, sse, sizeof(double) * n_img, cudaMemcpyDeviceToHost, c.stream));
      TMB_CUDA(cudaStreamSynchronize(c.stream));
    }
    c.arena.release(mk);
  });
}

int tmb_ttm(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, int mode, const double* m,
            int64_t rows, double* y) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    if (mode < 0 || mode >= order)
      throw Error(TMB_EINVAL, "mode " + std::to_string(mode) + " out of range for order-" + std::to_string(order) +
                                  " tensor");
    if (rows < 1) throw Error(TMB_EINVAL, "ttm factor must have at least one row");
    tmb::ttm_dev(c, x, to_dtype(dtype), d, mode, m, rows, 1, rows, y);
  });
}

int tmb_ttmc(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, const double* const* factors,
             const int64_t* frows, const int64_t* fcols, int skip, int transpose, int greedy, double* y) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    for (int n = 0; n < order; ++n) {
      if (n == skip) continue;
      const int64_t r = transpose ? frows[n] : fcols[n];
      if (r != d[n])
        throw Error(TMB_EINVAL, "mode " + std::to_string(n) + ": factor shape (" + std::to_string(frows[n]) + ", " +
                                    std::to_string(fcols[n]) + ") does not match tensor dim " + std::to_string(d[n]));
    }
    tmb::ttmc_dev(c, x, to_dtype(dtype), d, factors, frows, fcols, skip, transpose != 0, greedy != 0, y);
  });
}

int tmb_gram(tmb_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* g) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (rows < 1 || cols < 1) throw Error(TMB_EINVAL, "gram: empty matrix");
    tmb::mode_gram_dev(c, m, tmb::F64, Dims{rows, cols}, 0, g);
  });
}

int tmb_mirror_upper(tmb_ctx* ctx, double* g, int64_t n) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (n < 1) throw Error(TMB_EINVAL, "mirror_upper: empty matrix");
    tmb::mirror_upper(c, g, n, 1, 0);
  });
}

int tmb_mode_gram(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, int mode, double* g) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    if (mode < 0 || mode >= order)
      throw Error(TMB_EINVAL, "mode " + std::to_string(mode) + " out of range for order-" + std::to_string(order) +
                                  " tensor");
    tmb::mode_gram_dev(c, x, to_dtype(dtype), d, mode, g);
  });
}

int tmb_leading_eigvecs(tmb_ctx* ctx, const double* g, int64_t n, int64_t k, double* vecs, double* vals) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (n < 1) throw Error(TMB_EINVAL, "expected a square matrix");
    if (k < 1 || k > n)  // tensor.py:193-194
      throw Error(TMB_EINVAL, "k=" + std::to_string(k) + " out of range for " + std::to_string(n) + "x" +
                                  std::to_string(n) + " matrix");
    tmb::leading_eigvecs(c, g, n, k, vecs, vals);
  });
}

int tmb_tridiagonalize(tmb_ctx* ctx, const double* g, int64_t n, double* d, double* e) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (n < 3 || n > 8000) throw Error(TMB_EINVAL, "tridiagonalize: n must be in [3, 8000]");
    const size_t mk = c.arena.mark();
    double* A = tmb::alloc<double>(c, (size_t)n * n);
    double* hv = tmb::alloc<double>(c, (size_t)n * n);
    double* tau = tmb::alloc<double>(c, (size_t)n);
    double* band = tmb::alloc<double>(c, (size_t)n * (2 * tmb::SBR_B + 1));
    TMB_CUDA(cudaMemsetAsync(hv, 0, sizeof(double) * n * n, c.stream));
    TMB_CUDA(cudaMemsetAsync(tau, 0, sizeof(double) * n, c.stream));
    tmb::copy_d(c, A, g, n * n);
    tmb::sy2sb(c, A, n, hv, tau);
    tmb::band_rows(c, A, n, band);
    tmb::sb2st(c, band, n, d, e);
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    c.arena.release(mk);
  });
}

int tmb_sumsq(tmb_ctx* ctx, const void* x, int dtype, int64_t n, double* out) {
  return guard(ctx, [&](tmb::Ctx& c) { *out = tmb::sumsq(c, x, to_dtype(dtype), n); });
}

int tmb_resid_sumsq(tmb_ctx* ctx, const void* t, int dtype, const double* th, int64_t n, double* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const size_t mk = c.arena.mark();
    double* d = tmb::alloc<double>(c, 1);
    tmb::resid2_async(c, t, to_dtype(dtype), th, n, d);
    TMB_CUDA(cudaMemcpyAsync(c.host_pinned, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    *out = c.host_pinned[0];
    c.arena.release(mk);
  });
}

int tmb_axpy(tmb_ctx* ctx, int64_t n, double alpha, const double* x, double* y) {
  return guard(ctx, [&](tmb::Ctx& c) { tmb::axpy(c, n, alpha, x, y); });
}

int tmb_t_hosvd(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, const int64_t* ranks,
                int greedy, double* core, double* const* factors) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    const Dims r = check_ranks(d, ranks);
    tmb::t_hosvd_dev(c, x, to_dtype(dtype), d, r, greedy != 0, core, factors);
  });
}

int tmb_hooi_sweep(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, const int64_t* ranks,
                   const double* const* fin, int greedy, double* core, double* const* fout) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    const Dims r = check_ranks(d, ranks);
    tmb::hooi_sweep_dev(c, x, to_dtype(dtype), d, r, fin, greedy != 0, core, fout);
  });
}

int tmb_reconstruct(tmb_ctx* ctx, int order, const int64_t* ranks, const int64_t* dims, const double* core,
                    const double* const* factors, double* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    const Dims r = to_dims(order, ranks);
    tmb::reconstruct_dev(c, r, d, core, factors, out);
  });
}

int tmb_tucker_als(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, const int64_t* ranks,
                   const tmb_solve_cfg* cfg, double* core, double* const* factors, tmb_trace* trace) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    if (!cfg) throw Error(TMB_EINVAL, "null solve config");
    const Dims r = check_ranks(d, ranks);
    if (cfg->fit_tol <= 0 || cfg->pp_exit_tol <= 0) throw Error(TMB_EINVAL, "tolerances must be positive");
    if (cfg->max_sweeps < 0) throw Error(TMB_EINVAL, "max_sweeps must be >= 0");
    if (trace && trace->capacity < cfg->max_sweeps + 1) throw Error(TMB_EINVAL, "trace capacity < max_sweeps + 1");
    tmb::tucker_als_dev(c, x, to_dtype(dtype), d, r, *cfg, core, factors, trace);
  });
}

int tmb_solve_channels(tmb_ctx* ctx, const void* x, int dtype, const int64_t* dims, const int64_t* ranks,
                       const tmb_solve_cfg* cfg, double* const* cores, double* const* factors, tmb_trace* traces) {
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(4, dims);
    if (!cfg) throw Error(TMB_EINVAL, "null solve config");
    const Dims r = check_ranks(d, ranks);
    if (cfg->fit_tol <= 0 || cfg->pp_exit_tol <= 0) throw Error(TMB_EINVAL, "tolerances must be positive");
    if (cfg->max_sweeps < 0) throw Error(TMB_EINVAL, "max_sweeps must be >= 0");
    if (!cores || !factors) throw Error(TMB_EINVAL, "null output arrays");
    for (int ch = 0; ch < 3; ++ch)
      if (traces && traces[ch].capacity < cfg->max_sweeps + 1)
        throw Error(TMB_EINVAL, "trace capacity < max_sweeps + 1");
    const tmb::DType t = to_dtype(dtype);
    const int64_t P = tmb::prod(d, 0, 4);
    const size_t esz = t == tmb::F32 ? sizeof(float) : sizeof(double);
    for (int ch = 0; ch < 3; ++ch) {
      const void* xc = static_cast<const char*>(x) + (size_t)ch * (size_t)P * esz;
      tmb::tucker_als_dev(c, xc, t, d, r, *cfg, cores[ch], factors + 4 * ch, traces ? traces + ch : nullptr);
    }
  });
}

int tmb_color_f64_channels(tmb_ctx* ctx, const double* px, int64_t n_img, int64_t h, int64_t w, int space,
                           double* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    if (n_img < 0 || h < 0 || w < 0) throw Error(TMB_EINVAL, "negative image dimensions");
    tmb::color_f64_channels(c, px, n_img, h, w, space, out);
  });
}

int tmb_channels_to_rgb(tmb_ctx* ctx, const double* t, int64_t n_img, int64_t h, int64_t w, int space,
                        double* rgb) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space < TMB_SPACE_RGB || space > TMB_SPACE_IPT) throw Error(TMB_EINVAL, "unknown color space");
    if (n_img < 0 || h < 0 || w < 0) throw Error(TMB_EINVAL, "negative image dimensions");
    tmb::channels_to_rgb(c, t, n_img, h, w, space, rgb);
  });
}

int tmb_pp_operators(tmb_ctx* ctx, const void* x, int dtype, int order, const int64_t* dims, const int64_t* ranks,
                     const double* const* anchors, tmb_pp** out) {
  if (!out) return TMB_EINVAL;
  *out = nullptr;
  return guard(ctx, [&](tmb::Ctx& c) {
    const Dims d = to_dims(order, dims);
    const Dims r = check_ranks(d, ranks);
    if (order > 16 || !anchors) throw Error(TMB_EINVAL, "expected " + std::to_string(order) + " anchors");
    auto* h = new tmb_pp;
    h->device = c.device;
    try {
      tmb::pp_build(c, h->ops, x, to_dtype(dtype), d, r, anchors);
      TMB_CUDA(cudaStreamSynchronize(c.stream));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int tmb_pp_info(const tmb_pp* pp, int* order, int* contraction_count) {
  if (!pp) return TMB_EINVAL;
  if (order) *order = (int)pp->ops.dims.size();
  if (contraction_count) *contraction_count = pp->ops.count;
  return TMB_OK;
}

int tmb_pp_operator(const tmb_pp* pp, unsigned free_mask, const double** op_dev, int64_t* dims_out) {
  if (!pp || !op_dev) return TMB_EINVAL;
  const double* p = pp->ops.find(free_mask);
  if (!p) return TMB_EINVAL;
  *op_dev = p;
  if (dims_out) {
    const Dims d = tmb::pp_node_dims(pp->ops.dims, pp->ops.ranks, free_mask);
    for (size_t n = 0; n < d.size(); ++n) dims_out[n] = d[n];
  }
  return TMB_OK;
}

int tmb_pp_operator_copy(tmb_ctx* ctx, const tmb_pp* pp, unsigned free_mask, double* out) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (!pp || !out) throw Error(TMB_EINVAL, "null pp state or output");
    const double* p = pp->ops.find(free_mask);
    if (!p) throw Error(TMB_EINVAL, "no pp operator for free-mode mask " + std::to_string(free_mask));
    const Dims d = tmb::pp_node_dims(pp->ops.dims, pp->ops.ranks, free_mask);
    tmb::copy_d(c, out, p, tmb::prod(d, 0, (int)d.size()));
  });
}

int tmb_pp_set_deltas(tmb_ctx* ctx, tmb_pp* pp, const double* const* src, int src_are_factors, double* max_rel) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (!pp || !src) throw Error(TMB_EINVAL, "null pp state or inputs");
    const double m = tmb::pp_set_deltas(c, pp->ops, src, src_are_factors != 0);
    if (max_rel) *max_rel = m;
  });
}

int tmb_pp_sweep(tmb_ctx* ctx, tmb_pp* pp, double* core, double* const* factors, double* const* operands) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (!pp || !factors) throw Error(TMB_EINVAL, "null pp state or outputs");
    tmb::pp_sweep_dev(c, pp->ops, factors, core, operands);
  });
}

int tmb_pp_destroy(tmb_pp* pp) {
  if (!pp) return TMB_OK;
  cudaSetDevice(pp->device);
  delete pp;
  return TMB_OK;
}

int tmb_quantize_core(tmb_ctx* ctx, const double* core, int64_t n, int qp, int64_t* levels, double* step_host) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (qp < 0 || qp > 51) throw Error(TMB_EINVAL, "qp " + std::to_string(qp) + " out of range [0, 51]");
    const size_t mk = c.arena.mark();
    double* sc = tmb::alloc<double>(c, 2);
    if (n > 0) tmb::absmax_async(c, core, n, sc);
    else TMB_CUDA(cudaMemsetAsync(sc, 0, sizeof(double), c.stream));
    tmb::quant_step(c, sc, qp, sc + 1);
    tmb::quantize(c, core, n, sc + 1, levels);
    TMB_CUDA(cudaMemcpyAsync(c.host_pinned, sc + 1, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    if (step_host) *step_host = c.host_pinned[0];
    c.arena.release(mk);
  });
}

int tmb_dequantize(tmb_ctx* ctx, const int64_t* levels, int64_t n, double step, double* core) {
  return guard(ctx, [&](tmb::Ctx& c) { tmb::dequant(c, levels, n, step, core); });
}

int tmb_encode_stack_u8(tmb_ctx* ctx, const uint8_t* rgb, int64_t n_img, int64_t h, int64_t w, int space,
                        const int64_t* ranks, const tmb_solve_cfg* cfg, int qp, float* tensor, double* core,
                        double* const* factors, int64_t* levels, double* step_host, tmb_trace* trace,
                        double* rel_err_host) {
  return guard(ctx, [&](tmb::Ctx& c) {
    if (space != TMB_SPACE_YCBCR && space != TMB_SPACE_IPT && space != TMB_SPACE_RGB)
      throw Error(TMB_EINVAL, "unknown color space");
    if (qp < 0 || qp > 51) throw Error(TMB_EINVAL, "qp " + std::to_string(qp) + " out of range [0, 51]");
    if (!cfg) throw Error(TMB_EINVAL, "null solve config");
    const Dims d{h, w, 3, n_img};
    for (auto v : d)
      if (v < 1) throw Error(TMB_EINVAL, "all dimensions must be >= 1");
    const Dims r = check_ranks(d, ranks);
    tmb::color_u8(c, rgb, n_img, h, w, space, tensor);
    tmb::tucker_als_dev(c, tensor, tmb::F32, d, r, *cfg, core, factors, trace);
    const int64_t Pc = tmb::prod(r, 0, 4), P = tmb::prod(d, 0, 4);
    const size_t mk = c.arena.mark();
    double* sc = tmb::alloc<double>(c, 4);
    tmb::absmax_async(c, core, Pc, sc);
    tmb::quant_step(c, sc, qp, sc + 1);
    tmb::quantize(c, core, Pc, sc + 1, levels);
    if (rel_err_host) {  // K9: reconstruction fused with the residual norm (nothing written)
      tmb::reconstruct_resid_dev(c, r, d, core, factors, tensor, tmb::F32, sc + 2);
      tmb::sumsq_async(c, tensor, tmb::F32, P, sc + 3);
    }
    TMB_CUDA(cudaMemcpyAsync(c.host_pinned, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, c.stream));
    TMB_CUDA(cudaStreamSynchronize(c.stream));
    if (step_host) *step_host = c.host_pinned[1];
    if (rel_err_host) *rel_err_host = std::sqrt(c.host_pinned[2]) / std::sqrt(c.host_pinned[3]);
    c.arena.release(mk);
  });
}

}  // extern "C"
