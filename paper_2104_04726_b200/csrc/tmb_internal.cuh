// Internal declarations shared by the tmb kernels and the host-side solver.
// Layout conventions: tensors are F-order (mode 0 fastest, the
// reference's linearisation, tensor.py:1-13); factor matrices are column-major
// s_n x r_n (one eigenvector per contiguous column); all contraction
// arithmetic accumulates in fp64.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tmb.h"

namespace tmb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TMB_CUDA(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::tmb::Error(TMB_ECUDA, std::string(#x ": ") + cudaGetErrorString(e_));    \
  } while (0)

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(TMB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Bump arena over retained device chunks: no cudaMalloc inside steady-state loops.
class Arena {
 public:
  ~Arena();
  void* alloc(size_t bytes);
  size_t mark() const;
  void release(size_t mark);
  void free_all();
  size_t capacity() const;
  size_t peak() const { return peak_; }  // high-water mark of bytes in use
  void reserve(size_t bytes);            // one retained chunk of at least `bytes`

 private:
  struct Chunk { char* p; size_t cap; size_t used; };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0;
  size_t peak_ = 0;
};

// Per-family launch timing (CUDA events on the context stream), enabled by the
// benchmark to measure the dominant kernel's live launch durations.
struct KernelTimes {
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec { int tag; size_t a, b; double work; };
  std::vector<Rec> recs;
};
enum TimerTag { TAG_GEMM = 0, TAG_SYTRD, TAG_TRIDIAG, TAG_COLOR, TAG_EIG_GEMM, TAG_OZAKI, TAG_COUNT };

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  Arena arena;
  double* host_pinned = nullptr;   // small D2H staging for scalars
  int64_t launches = 0;            // kernels launched by this context
  int coop_blocks = 0;             // resident blocks for cooperative kernels
  bool timing = false;
  KernelTimes kt;
  double work[TAG_COUNT] = {0};    // algorithmic flops/bytes attributed per tag
  int gemm_tag = TAG_GEMM;         // TAG_EIG_GEMM while inside the eigen-solver
  // Ozaki digit planes of a tensor operand kept for the rest of one solve (tucker_als
  // re-splits the same raw tensor identically every sweep otherwise): buffers from the
  // solve's arena frame, registered by ozaki_cache_begin, filled on first use.
  struct OzSlot {
    const void* x = nullptr;
    int64_t L = 0, K = 0, R = 0;
    int tx = -1;
    int8_t* sx = nullptr;
    int* ex = nullptr;
    bool valid = false;
  };
  OzSlot ozs[2];
  void oz_clear() { for (auto& z : ozs) z = OzSlot{}; }
};

// RAII: records an event pair around the launches in its scope (if enabled)
// and attributes `work` algorithmic units (flops or bytes) to the tag.
class Timed {
 public:
  Timed(Ctx& c, int tag, double work);
  ~Timed();
 private:
  Ctx& c_;
  int tag_;
  size_t a_ = 0;
  double work_;
};

template <typename T>
T* alloc(Ctx& c, size_t n) { return static_cast<T*>(c.arena.alloc(n * sizeof(T))); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Per-(device, kernel) attribute / occupancy caches (devcache.cu): raise the
// kernel's dynamic shared-memory limit to at least `bytes` on c.device once;
// resident blocks per SM for (kernel, threads, smem) on c.device.
void set_smem_attr(Ctx& c, const void* fn, size_t bytes);
int blocks_per_sm(Ctx& c, const void* fn, int threads, size_t smem);

// ---------------------------------------------------------------- GEMM (k_gemm.cu)
enum DType { F32 = 0, F64 = 1 };

// C[b](m,n) = alpha * sum_{k1,k2} A[b](m,k1,k2) B[b](k1,k2,n) + beta * C[b](m,n)
// with arbitrary element strides; fp64 accumulation on the DMMA pipe.
struct GemmDesc {
  int64_t M = 0, N = 0, K1 = 0, K2 = 1;
  int batch = 1;
  const void* A = nullptr; DType ta = F64; int64_t sAm = 0, sAk1 = 0, sAk2 = 0, sAb = 0;
  const void* B = nullptr; DType tb = F64; int64_t sBn = 0, sBk1 = 0, sBk2 = 0, sBb = 0;
  double* C = nullptr; int64_t sCm = 0, sCn = 0, sCb = 0;
  double alpha = 1.0, beta = 0.0;
  bool syrk_upper = false;   // only tiles touching the upper triangle (caller mirrors)
  int splits = 0;            // 0 = auto
};
void gemm(Ctx& c, const GemmDesc& d);
void mirror_upper(Ctx& c, double* g, int64_t n, int batch, int64_t sb);

// ---------------------------------------------------------------- small kernels (k_small.cu)
void small_ttm(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t Rr,
               const double* m, int64_t r, int64_t sMr, int64_t sMk, double* y);
// two consecutive small-mode TTMs (modes m, m+1) in one pass, bitwise equal to
// two small_ttm calls; false (nothing launched) outside its size limits
bool small_ttm2(Ctx& c, const void* x, DType tx, int64_t L, int64_t K1, int64_t K2, int64_t Rr, const double* m1,
                int64_t r1, int64_t s1r, int64_t s1k, const double* m2, int64_t r2, int64_t s2r, int64_t s2k,
                double* y);
// the same two products fused with sum (t - y)^2 (K9 epilogue: y is never written);
// false (nothing launched) outside small_ttm2's limits
bool small_ttm2_resid(Ctx& c, const double* x, int64_t L, int64_t K1, int64_t K2, int64_t Rr, const double* m1,
                      int64_t r1, int64_t s1r, int64_t s1k, const double* m2, int64_t r2, int64_t s2r, int64_t s2k,
                      const void* t, DType tt, double* out_dev);
void small_gram(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t Rr, double* g);
double sumsq(Ctx& c, const void* x, DType tx, int64_t n);           // sync D2H
void sumsq_async(Ctx& c, const void* x, DType tx, int64_t n, double* out_dev);
void absmax_async(Ctx& c, const double* x, int64_t n, double* out_dev);
void quantize(Ctx& c, const double* core, int64_t n, const double* step_dev, int64_t* levels);
void quant_step(Ctx& c, const double* amax_dev, int qp, double* step_dev);
void sign_fix(Ctx& c, double* v, int64_t n, int64_t k);
void diff_norms(Ctx& c, const double* a, const double* b, int64_t n, double* out2_dev);
void copy_d(Ctx& c, double* dst, const double* src, int64_t n);
void scale_identity_combo(Ctx& c, const double* w, int64_t n, double a, double b, double* out);
void maxabs_offidentity(Ctx& c, const double* w, int64_t n, double* out_dev);
void convert_f32_f64(Ctx& c, const float* s, double* d, int64_t n);
void dequant(Ctx& c, const int64_t* lv, int64_t n, double step, double* out);
void axpy(Ctx& c, int64_t n, double alpha, const double* x, double* y);
void resid2_async(Ctx& c, const void* t, DType tt, const double* that, int64_t n, double* out_dev);

// ---------------------------------------------------------------- eigensolvers (k_eig.cu)
// Dominant-k eigenpairs of a symmetric n x n (column-major) matrix, eigenvalues
// nonincreasing, columns sign-fixed (tensor.py:183-209). g is not modified.
void leading_eigvecs(Ctx& c, const double* g, int64_t n, int64_t k, double* vecs, double* vals);
// Row-partitioned cooperative tridiagonalisation for n <= 2048 (k_sytrd_rows.cu);
// false if n is out of its range.
bool sytrd_rows(Ctx& c, double* A, int64_t n, int64_t k_end, double* d, double* e, double* tau, double* hv,
                double* pbuf);
// Shared-memory-resident tridiagonalisation of an n x n symmetric block stored with leading
// dimension ld (d, e, tau, hv offset to the block; hv with the same ld); steps 0 .. k_end-1,
// the rest left in A for a tail kernel. resume: reflector 0 (hv column 0, tau[0], d[0], e[0])
// was computed by the kernel that ran the earlier steps (the column kernel stopped there).
// False if the block's columns do not fit shared memory.
bool sytrd_smem(Ctx& c, double* A, int64_t n, int64_t k_end, double* d, double* e, double* tau, double* hv,
                double* pbuf, int64_t ld, int resume);
// Cluster-resident tridiagonalisation of the trailing block from step K0 (k_sytrd_tail.cu).
int64_t sytrd_tail_capacity(Ctx& c);
void sytrd_tail(Ctx& c, double* A, int64_t n, int64_t K0, double* d, double* e, double* tau, double* hv);
// Single-CTA tridiagonalisation of a trailing block of <= sytrd_tail1_max() from step K0 (k_sytrd_tail1.cu).
int64_t sytrd_tail1_max();
void sytrd_tail1(Ctx& c, double* A, int64_t n, int64_t K0, double* d, double* e, double* tau, double* hv);

// ---------------------------------------------------------------- two-stage tridiagonalisation (k_twostage.cu)
constexpr int SBR_B = 32;  // half-bandwidth of the intermediate band matrix
// stage 1: symmetric A (n x n, column-major) -> band of half-bandwidth SBR_B in place
// (entries outside the band are left undefined); reflector of column c in hv column c
// (zero above its first row; hv and tau must be zeroed by the caller)
void sy2sb(Ctx& c, double* A, int64_t n, double* hv, double* tau);
// the band of A as full rows: band[r * (2 SBR_B + 1) + (col - r + SBR_B)]
void band_rows(Ctx& c, const double* A, int64_t n, double* band);
// stage 2: band -> tridiagonal (d: n diagonal, e: n-1 subdiagonal)
void sb2st(Ctx& c, const double* band, int64_t n, double* d, double* e);
// unit eigenvectors of the band matrix for the k eigenvalues vals (n x k, column-major)
void band_invit(Ctx& c, const double* band, int64_t n, int64_t k, const double* vals, double* z);

// ---------------------------------------------------------------- colour (k_color.cu)
void color_u8(Ctx& c, const uint8_t* rgb, int64_t n_img, int64_t h, int64_t w, int space, float* out,
              bool channel_major = false);
void color_f64(Ctx& c, const double* rgb, int64_t npx, int space, double* out);
void color_inv_f64(Ctx& c, const double* px, int64_t npx, int space, double* out, int64_t* n_clamped);
// codec float64 path: interleaved (img, h, w, 3) pixels -> three F-order (h, w, E, V) channel tensors
void color_f64_channels(Ctx& c, const double* px, int64_t n_img, int64_t h, int64_t w, int space, double* out);
// inverse: three (h, w, E, V) channel tensors -> to_rgb -> interleaved (img, h, w, 3)
void channels_to_rgb(Ctx& c, const double* t, int64_t n_img, int64_t h, int64_t w, int space, double* rgb);
// decode: coding-space F-order stack -> RGB (optional interleaved output) and the
// per-image SSE in 8-bit units vs the original u8 images (rgb may be null)
void decode_sse(Ctx& c, const double* t, int64_t n_img, int64_t h, int64_t w, int space, const uint8_t* rgb,
                double* out_rgb, double* sse_dev);

// ---------------------------------------------------------------- Ozaki TTM on tcgen05 (k_ozaki.cu)
// y = x x_n mat over the GEMM view rows (i < L, l < R), K = dims[n], N = rows of mat
// (mat(r, k) at mat[r sMr + k sMk]); fp64-equivalent via int8 digit products.
bool ozaki_enabled();
// register (and allocate from the current arena frame) a digit-plane cache slot for the
// tensor operand x viewed as (L, K, R) with K contracted; ozaki_ttm reuses it when asked
// for the same operand again before c.oz_clear()
void ozaki_cache_slot(Ctx& c, int slot, const void* x, DType tx, int64_t L, int64_t K, int64_t R);
void ozaki_ttm(Ctx& c, const void* x, DType tx, int64_t L, int64_t K, int64_t R, const double* mat, int64_t N,
               int64_t sMr, int64_t sMk, double* y);

// ---------------------------------------------------------------- latent block bytes (k_latent.cu)
// zigzag + LEB128 varints of int64 levels (entropy.py:55-111); returns the byte count
int64_t varint_encode(Ctx& c, const int64_t* levels, int64_t n, uint8_t* out, int64_t cap);
// inverse (entropy.py:88-117); returns the bytes consumed, throws TMB_EINVAL when corrupt
int64_t varint_decode(Ctx& c, const uint8_t* in, int64_t nbytes, int64_t count, int64_t* levels);

}  // namespace tmb
