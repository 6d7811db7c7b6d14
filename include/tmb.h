/* tmb.h -- C ABI of the B200 Tucker-ALS (HOOI) hot path.
 *
 * This is the drop-in boundary for the Python API of the reference package
 * `tmcodec` (arXiv 2104.04726 coder). Each entry point names the reference
 * function it replaces (paths relative to /root/reference/pkg/src/tmcodec/).
 * The reference has no compiled FFI for this path -- its boundary is the
 * Python package surface (__init__.py:3-62) -- so the binding a maintainer
 * adds is the ctypes shim shown in INTEGRATION.md.
 *
 * Conventions
 *  - Every pointer argument named *_dev is a DEVICE pointer owned by the caller
 *    (the library only owns a per-context workspace arena).
 *  - Tensors are dense, F-order (mode 0 fastest): the reference linearisation
 *    (tensor.py:1-13, DenseTensor.data tensor.py:74-78).
 *  - Matrices (factors, Grams, eigenvectors) are column-major.
 *  - All arithmetic accumulates in float64; tensors may be given as float32
 *    (TMB_F32, the device format of the colour-converted stack) or float64.
 *  - Return value: TMB_OK or an error code; tmb_last_error() has the text.
 *    TMB_EINVAL messages reproduce the reference ValueError wording.
 *  - A context is bound to one device and one CUDA stream; contexts are not
 *    internally synchronised (one per host thread). Calls are stream-ordered;
 *    functions that return host scalars synchronise the stream.
 */
#ifndef TMB_H_
#define TMB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TMB_OK = 0, TMB_EINVAL = 1, TMB_ENUMERIC = 2, TMB_ECUDA = 3, TMB_ENOTIMPL = 4 };
enum { TMB_SPACE_RGB = 0, TMB_SPACE_YCBCR = 1, TMB_SPACE_IPT = 2 };
enum { TMB_F32 = 0, TMB_F64 = 1 };
enum { TMB_KIND_INIT = 0, TMB_KIND_STANDARD = 1, TMB_KIND_PP = 2 };

typedef struct tmb_ctx tmb_ctx;

/* SolveConfig (tucker.py:74-95); ranks are passed separately. */
typedef struct {
  int max_sweeps;
  double fit_tol;
  double pp_enter_tol;
  double pp_exit_tol;
  int sequential_reduction; /* 1 = ascending contraction order, 0 = greedy */
} tmb_solve_cfg;

/* SolveTrace / SweepRecord (tucker.py:98-113). Arrays are caller-owned HOST
 * memory of length `capacity` (>= max_sweeps + 1). */
typedef struct {
  int capacity;
  int n_records;
  int converged;
  int best_index;   /* record index of the returned model */
  int* kind;        /* TMB_KIND_* */
  double* fit;
  double* max_change; /* NaN for the init record */
} tmb_trace;

/* ---- context ---------------------------------------------------------- */
int tmb_ctx_create(int device, void* cuda_stream, tmb_ctx** out);
int tmb_ctx_destroy(tmb_ctx* ctx);
int tmb_ctx_set_stream(tmb_ctx* ctx, void* cuda_stream);
const char* tmb_last_error(const tmb_ctx* ctx);
int64_t tmb_launch_count(const tmb_ctx* ctx); /* kernels launched so far */
/* Workspace pool (caller owns every input/output buffer; the
 * library owns one per-context pool of retained device chunks). Reports the
 * reserved bytes and the high-water mark of bytes in use so far; reserve()
 * replaces a smaller pool by one chunk of `bytes` (call between solves, e.g.
 * with the peak of a first solve, so no later call allocates). No reference
 * counterpart: the reference's numpy arrays are allocated per call. */
int tmb_workspace_size(const tmb_ctx* ctx, int64_t* reserved_bytes, int64_t* peak_bytes);
int tmb_workspace_reserve(tmb_ctx* ctx, int64_t bytes);
/* Launch timing by kernel family (CUDA events on the context stream), used by
 * bench.py for the roofline: tags 0 DMMA GEMM (TTM/Gram), 1 tridiagonalisation,
 * 2 bisection+twisted vectors, 3 colour, 4 DMMA GEMMs inside the eigen-solver, 5 Ozaki int8
 * tcgen05 TTM (digit split + GEMM; work in fp64-equivalent flops). tmb_timing(ctx, 1)
 * resets and enables; tmb_timing_read returns launches, total ms and the
 * algorithmic work (flops, or bytes for colour) attributed to the tag. */
enum { TMB_TAG_GEMM = 0, TMB_TAG_SYTRD = 1, TMB_TAG_TRIDIAG = 2, TMB_TAG_COLOR = 3, TMB_TAG_EIG_GEMM = 4, TMB_TAG_OZAKI = 5 };
int tmb_timing(tmb_ctx* ctx, int enable);
int tmb_timing_read(tmb_ctx* ctx, int tag, int64_t* count, double* ms, double* work);
int tmb_version(void);

/* ---- colour (color.py) ------------------------------------------------ */
/* n_img interleaved sRGB u8 images (h x w x 3, row-major, the PNG sample
 * order of sceneio.read_image) -> float32 F-order tensor (h, w, 3, n_img) in
 * the coding space: rgb_to_ycbcr (color.py:111-119) / rgb_to_ipt
 * (color.py:145-158) of u8/255 (sceneio.py:87), stacked as in SURVEY §8.0. */
int tmb_color_u8(tmb_ctx* ctx, const uint8_t* rgb_dev, int64_t n_img, int64_t h, int64_t w,
                 int space, float* tensor_dev);
/* The same colour transform into the reference codec's per-channel layout:
 * three float32 F-order (h, w, E, V) tensors back to back (channel c at
 * tensor_dev + c*h*w*n_img), i.e. stack_to_tensor(stack, c) for c = 0, 1, 2
 * (sceneio.py:38, 191-199) of the converted stack (codec.py:389). */
int tmb_color_u8_channels(tmb_ctx* ctx, const uint8_t* rgb_dev, int64_t n_img, int64_t h, int64_t w,
                          int space, float* tensor_dev);
/* Pixelwise float64 transforms on npx interleaved pixels (ColorImage.pixels):
 * to_coding_space (color.py:185-194) and to_rgb (color.py:197-205). */
int tmb_color_f64(tmb_ctx* ctx, const double* px_dev, int64_t npx, int space, double* out_dev);
int tmb_color_inv_f64(tmb_ctx* ctx, const double* px_dev, int64_t npx, int space,
                      double* out_dev, int64_t* n_clamped_host);

/* The latent codec's float64 colour path: n_img interleaved float64 RGB images
 * (n_img, h, w, 3) -- the scene's ColorImage.pixels in (view, exposure) order --
 * through to_coding_space (color.py:185-194, codec.py:389) straight into the
 * per-channel layout of stack_to_tensor (sceneio.py:191-199): three float64
 * F-order (h, w, E, V) tensors back to back (channel c at out + c*h*w*n_img).
 * tmb_channels_to_rgb is the decode side's inverse (tensor_to_stack,
 * sceneio.py:202-226, then to_rgb per image, codec.py:466-468). */
int tmb_color_f64_channels(tmb_ctx* ctx, const double* px_dev, int64_t n_img, int64_t h, int64_t w, int space,
                           double* tensor_dev);
int tmb_channels_to_rgb(tmb_ctx* ctx, const double* tensor_dev, int64_t n_img, int64_t h, int64_t w, int space,
                        double* rgb_out_dev);

/* Decode side: tensor_dev is a reconstructed coding-space
 * stack (float64 F-order h x w x 3 x n_img: reconstruct(dequantize(q)),
 * codec.py:446-447); every pixel goes through to_rgb (color.py:197-205).
 * rgb_out_dev (nullable) receives interleaved float64 RGB images (n_img, h, w,
 * 3). With rgb_dev (nullable; the original u8 images, same layout as
 * tmb_color_u8's input) sse_host[n_img] receives each image's sum of squared
 * differences in 8-bit units, sum((u8/255*255 - 255*rgb)^2): metrics.mse
 * (metrics.py:16-23) times 3*h*w, as scene_psnr evaluates it (:41-76). */
int tmb_decode_sse(tmb_ctx* ctx, const double* tensor_dev, int64_t n_img, int64_t h, int64_t w, int space,
                   const uint8_t* rgb_dev, double* rgb_out_dev, double* sse_host);

/* ---- tensor kernels (tensor.py) ---------------------------------------- */
/* ttm (tensor.py:111-123): y = x x_mode m, m column-major rows x dims[mode]. */
int tmb_ttm(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims, int mode,
            const double* m_dev, int64_t rows, double* y_dev);
/* ttmc (tensor.py:138-173): factors[n] column-major with frows[n] x fcols[n];
 * applied as factors[n]^T when transpose != 0. skip < 0 means none. */
int tmb_ttmc(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
             const double* const* factors_dev, const int64_t* frows, const int64_t* fcols,
             int skip, int transpose, int greedy, double* y_dev);
/* gram (tensor.py:176-180): g = m m^T for column-major rows x cols m, exactly
 * symmetric (upper triangle computed, mirrored). */
int tmb_gram(tmb_ctx* ctx, const double* m_dev, int64_t rows, int64_t cols, double* g_dev);
/* g <- triu(g) + triu(g, 1)^T for a column-major n x n g (the exact symmetry
 * of gram, tensor.py:176-180), for Grams assembled from separately computed
 * blocks (the row-sharded solver's mode-0 Gram). */
int tmb_mirror_upper(tmb_ctx* ctx, double* g_dev, int64_t n);
/* gram(unfold(x, mode)) without materialising the unfolding. */
int tmb_mode_gram(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
                  int mode, double* g_dev);
/* leading_eigvecs (tensor.py:183-209): dominant k eigenpairs of the symmetric
 * n x n g, eigenvalues nonincreasing, each column sign-fixed so its first
 * max-|entry| is positive. vecs column-major n x k. */
int tmb_leading_eigvecs(tmb_ctx* ctx, const double* g_dev, int64_t n, int64_t k,
                        double* vecs_dev, double* vals_dev);
/* The tridiagonal form T = Q^T g Q behind leading_eigvecs for large n (the
 * two-stage reduction: dense -> band of half-bandwidth 32 -> tridiagonal; the
 * reference reaches the same T inside eigh, tensor.py:195). d: n diagonal,
 * e: n-1 subdiagonal entries (device). 3 <= n <= 8000 (the band of stage 2 lives in one
 * 16-CTA thread-block cluster). */
int tmb_tridiagonalize(tmb_ctx* ctx, const double* g_dev, int64_t n, double* d_dev, double* e_dev);
/* fro_norm^2 (tensor.py:212-214), deterministic fp64 reduction; host result. */
int tmb_sumsq(tmb_ctx* ctx, const void* x_dev, int dtype, int64_t n, double* out_host);

/* sum((t - t_hat)^2) for t (dtype) and float64 t_hat: the residual of
 * fit(method="residual") (tucker.py:186-188); host result. */
int tmb_resid_sumsq(tmb_ctx* ctx, const void* t_dev, int dtype, const double* that_dev, int64_t n,
                    double* out_host);
/* y += alpha * x (float64): the PP operand accumulation (tucker.py:268-282). */
int tmb_axpy(tmb_ctx* ctx, int64_t n, double alpha, const double* x_dev, double* y_dev);

/* ---- Tucker solver (tucker.py) ------------------------------------------ */
/* t_hosvd (tucker.py:130-148). core F-order (ranks), factors[n] column-major. */
int tmb_t_hosvd(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
                const int64_t* ranks, int greedy, double* core_dev, double* const* factors_dev);
/* hooi_sweep (tucker.py:151-163) from factors_in to factors_out (may alias). */
int tmb_hooi_sweep(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
                   const int64_t* ranks, const double* const* factors_in_dev, int greedy,
                   double* core_dev, double* const* factors_out_dev);
/* reconstruct (tucker.py:166-171): out F-order dims. */
int tmb_reconstruct(tmb_ctx* ctx, int order, const int64_t* ranks, const int64_t* dims,
                    const double* core_dev, const double* const* factors_dev, double* out_dev);
/* tucker_als (tucker.py:331-397): full driver incl. trace, convergence,
 * best-of selection and the pairwise-perturbation phase (PP operators from a
 * memoised dimension tree, first-order sweeps with the entry deltas, exact
 * core re-projection, fit-dip rejection and anchor refresh; tucker.py:199-311,
 * 359-387). */
int tmb_tucker_als(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
                   const int64_t* ranks, const tmb_solve_cfg* cfg, double* core_dev,
                   double* const* factors_dev, tmb_trace* trace);

/* _solve_channels (codec.py:366-374): the latent path's three per-channel
 * tucker_als solves in one call. x_dev holds the three (dims) tensors back to
 * back (channel c at x_dev + c*prod(dims) elements of dtype); cores_dev[c],
 * factors_dev[4c + n] and traces[c] (each may be NULL) receive channel c's
 * model and trace. Same validation and error text as tmb_tucker_als. */
int tmb_solve_channels(tmb_ctx* ctx, const void* x_dev, int dtype, const int64_t* dims, const int64_t* ranks,
                       const tmb_solve_cfg* cfg, double* const* cores_dev, double* const* factors_dev,
                       tmb_trace* traces);

/* Pairwise perturbation (tucker.py:199-311) as a native handle owning the
 * dimension-tree operators on the device.
 *  tmb_pp_operators : pp_operators (tucker.py:222-265), the memoised dimension
 *                     tree (parent = re-add the largest contracted mode, so
 *                     every node is an ascending contraction; 13 contractions
 *                     for N = 4), anchors[n] column-major dims[n] x ranks[n].
 *  tmb_pp_operator  : device pointer + dims of the operator whose free modes
 *                     are `free_mask` (op_single: 1<<n, pair(i, n): 1<<i|1<<n),
 *                     owned by the handle.
 *  tmb_pp_operator_copy: the same operator copied into a caller buffer.
 *  tmb_pp_set_deltas: PPState.set_current (src_are_factors = 1: d = f - a) or
 *                     PPState.deltas = src (0); returns max_rel_delta
 *                     (tucker.py:212-219).
 *  tmb_pp_sweep     : pp_sweep (tucker.py:285-311) from the stored deltas:
 *                     factors_dev[n] receive the new factors, core_dev (nullable)
 *                     the pp core estimate, operands_dev[n] (nullable array /
 *                     entries) the first-order operands. */
typedef struct tmb_pp tmb_pp;
int tmb_pp_operators(tmb_ctx* ctx, const void* x_dev, int dtype, int order, const int64_t* dims,
                     const int64_t* ranks, const double* const* anchors_dev, tmb_pp** out);
int tmb_pp_info(const tmb_pp* pp, int* order, int* contraction_count);
int tmb_pp_operator(const tmb_pp* pp, unsigned free_mask, const double** op_dev, int64_t* dims_out);
int tmb_pp_operator_copy(tmb_ctx* ctx, const tmb_pp* pp, unsigned free_mask, double* out_dev);
int tmb_pp_set_deltas(tmb_ctx* ctx, tmb_pp* pp, const double* const* src_dev, int src_are_factors,
                      double* max_rel_delta_host);
int tmb_pp_sweep(tmb_ctx* ctx, tmb_pp* pp, double* core_dev, double* const* factors_dev,
                 double* const* operands_dev);
int tmb_pp_destroy(tmb_pp* pp);

/* ---- codec (codec.py) --------------------------------------------------- */
/* quantize_core (codec.py:114-134): int64 levels, step returned to host. */
int tmb_quantize_core(tmb_ctx* ctx, const double* core_dev, int64_t n, int qp,
                      int64_t* levels_dev, double* step_host);
/* dequantize core part (codec.py:137-148): core = levels * step. */
int tmb_dequantize(tmb_ctx* ctx, const int64_t* levels_dev, int64_t n, double step,
                   double* core_dev);

/* Latent-block level bytes: encode_ints / decode_ints (entropy.py:55-117) on
 * the device -- zigzag map + LEB128 varints, low 7-bit group first. Encode
 * writes at most cap bytes to out_dev and returns the byte count (EINVAL if
 * cap is too small); decode reads count values and returns the bytes consumed
 * (EINVAL "varint stream truncated ..." / "varint longer than 10 bytes"). */
int tmb_varint_encode(tmb_ctx* ctx, const int64_t* levels_dev, int64_t n, uint8_t* out_dev, int64_t cap,
                      int64_t* nbytes_host);
int tmb_varint_decode(tmb_ctx* ctx, const uint8_t* in_dev, int64_t nbytes, int64_t count, int64_t* levels_dev,
                      int64_t* used_host);

/* Entropy stage tag 1 (entropy.py:37-52): the reference's adaptive order-0
 * range coder (_kernels_py.py:24-109, _kernels.pyx:27-141), byte-identical, on
 * HOST buffers (serial byte work after the device path; no context needed).
 * tmb_rc_bound gives an output capacity sufficient for n input bytes; encode
 * returns the byte count in *n_out (EINVAL if cap is too small); decode reads
 * exactly n symbols (missing input bytes read as 0, as in the reference). */
int tmb_rc_bound(int64_t n, int64_t* cap);
int tmb_rc_encode(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap, int64_t* n_out);
int tmb_rc_decode(const uint8_t* in, int64_t n_in, int64_t n, uint8_t* out);

/* ---- fused hot path ------------------------------------------------------
 * One stack end to end: u8 images -> colour (tmb_color_u8) -> tucker_als ->
 * quantize_core -> reconstruct + relative error ||t - t_hat|| / ||t||.
 * tensor_dev (float32, h*w*3*n_img) receives the coding-space tensor;
 * rel_err_host may be NULL to skip the reconstruction. */
int tmb_encode_stack_u8(tmb_ctx* ctx, const uint8_t* rgb_dev, int64_t n_img, int64_t h, int64_t w,
                        int space, const int64_t* ranks, const tmb_solve_cfg* cfg, int qp,
                        float* tensor_dev, double* core_dev, double* const* factors_dev,
                        int64_t* levels_dev, double* step_host, tmb_trace* trace,
                        double* rel_err_host);

#ifdef __cplusplus
}
#endif
#endif /* TMB_H_ */
