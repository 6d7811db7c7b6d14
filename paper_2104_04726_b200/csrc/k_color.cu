// Colour transforms (color.py). The hot-path kernel reads interleaved u8 sRGB
// images and writes the coding-space tensor directly in the solver's F-order
// layout (h fastest), transposing 32x32 pixel tiles through shared memory so
// both the byte reads and the float writes are coalesced. It is HBM-bound:
// 3 B read + 12 B written per pixel.
//
// Arithmetic is fp64 in the reference's operation order without FMA
// contraction (__dmul_rn/__dadd_rn), then rounded once to fp32, so the Y'CbCr
// tensor is bit-identical to fp32(reference f64 colour). The IPT path uses a
// host-built 256-entry EOTF table (the u8 codes are exact) and CUDA pow for
// the 0.43 power; its matrix products follow the reference's 3x3 order.
#include <mutex>
#include <type_traits>

#include "tmb_internal.cuh"

namespace tmb {
namespace {

struct ColorConst {
  double eotf[256];
  double rgb2xyz[9];
  double xyz2lms[9];
  double lms2ipt[9];
  double xyz2rgb[9];
  double lms2xyz[9];
  double ipt2lms[9];
  double lin2lms[9];  // xyz2lms . rgb2xyz, for the u8 fast path
  double plog[6];     // log2(1 + r) = r (plog[5] + r (plog[4] + ... + r plog[0]))
  double pexp[7];     // 0.43, ln 2, then e^t coefficients 1/720 .. 1/2
};
__constant__ ColorConst cc;

constexpr double KR = 0.299, KG = 0.587, KB = 0.114;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void ycbcr(double r, double g, double b, double* o) {
  // color.py:116-118
  const double y = add(add(mul(KR, r), mul(KG, g)), mul(KB, b));
  const double cb = add(__ddiv_rn(mul(0.5, sub(b, y)), 1.0 - KB), 0.5);
  const double cr = add(__ddiv_rn(mul(0.5, sub(r, y)), 1.0 - KR), 0.5);
  o[0] = fmin(fmax(y, 0.0), 1.0);
  o[1] = fmin(fmax(cb, 0.0), 1.0);
  o[2] = fmin(fmax(cr, 0.0), 1.0);
}

__device__ __forceinline__ void mat3(const double* m, const double* v, double* o) {
  for (int i = 0; i < 3; ++i) o[i] = add(add(mul(v[0], m[3 * i]), mul(v[1], m[3 * i + 1])), mul(v[2], m[3 * i + 2]));
}

__device__ __forceinline__ double spow(double v, double p) {
  // color.py:141-142 sign(v) * |v|**p
  const double a = pow(fabs(v), p);
  return v > 0.0 ? a : (v < 0.0 ? -a : 0.0);
}

// sign(v) |v|^0.43 as exp2(0.43 log2 |v|): a few ulp in fp64 (vs pow's ~1), far
// cheaper; the u8 path's fp32 output stays bit-identical to the reference on all
// 2^24 RGB triples (tests/test_gpu_api.py::test_colour_u8_exhaustive)
__device__ __forceinline__ double spow043(double v) {
  const double a = exp2(0.43 * log2(fabs(v)));
  return v > 0.0 ? a : (v < 0.0 ? -a : 0.0);
}

// |v|^0.43 for the u8 IPT path from 128-entry tables + short polynomials, all
// fp64 (~20 DFMA-class ops instead of the ~70 of CUDA's log2 + exp2):
//   log2 a = e + lc_j + log2(1 + r) for a = m 2^e, r = m invc_j - 1 (|r| < 2^-8),
//            lc_j = -log2(invc_j), j = the top 7 bits of m,
//            log2(1 + r) by its degree-6 Taylor polynomial (truncation < 2^-56 |r|);
//   2^z    = 2^k 2^(i/128) e^(g ln 2), z = k + i/128 + g, g < 2^-7, degree-6 polynomial.
// Error ~2e-15 relative (the same class as exp2(0.43 log2)); the fp32 outputs are
// checked bit-identical to the reference on all 2^24 u8 triples
// (tests/test_gpu_api.py::test_colour_u8_exhaustive). The tables are staged in
// shared memory by the kernel.
constexpr int PT = 128;
struct PowTab {
  double invc[PT];   // RN(1 / (1 + (j + 0.5) / 128))
  double lc[PT];     // -log2(invc[j]) (so log2 m = lc + log2(m invc) exactly in real arithmetic)
  double e2[PT];     // 2^(j / 128)
};
__device__ PowTab g_powtab;

__device__ __noinline__ double pow043_slow(double v) {  // zero / subnormal |v| (never on u8 inputs)
  const double a = fabs(v);
  if (a == 0.0) return 0.0;
  const double y = exp2(0.43 * log2(a));
  return v > 0.0 ? y : -y;
}

__device__ __forceinline__ double pow043_tab(double v, const double* invc, const double* lc, const double* e2) {
  // polynomial coefficients and other fp64 constants come from the constant bank
  // (cc.*): as immediates each use re-materialised a 64-bit value through two
  // uniform-register moves per pixel
  const double a = fabs(v);
  const long long bits = __double_as_longlong(a);
  const int eb = (int)(bits >> 52);
  if (eb == 0) return pow043_slow(v);  // zero / subnormal
  const int j = (int)((bits >> 45) & (PT - 1));
  const double m = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double r = fma(m, invc[j], -1.0);
  double p = cc.plog[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) p = fma(p, r, cc.plog[i]);
  const double lg = ((double)(eb - 1023) + lc[j]) + p * r;
  const double z = cc.pexp[0] * lg;                 // 0.43 log2 a
  const double kf = floor(z);
  const double f = z - kf;                          // exact, in [0, 1)
  const double fi = floor(f * (double)PT);
  const double g = fma(fi, -1.0 / PT, f);           // exact, in [0, 1/128)
  const double t = g * cc.pexp[1];                  // g ln 2
  double q = cc.pexp[2];
#pragma unroll
  for (int i = 3; i < 7; ++i) q = fma(q, t, cc.pexp[i]);
  q = fma(q, t, 1.0);
  q = fma(q, t, 1.0);
  const double y = e2[(int)fi] * q * __longlong_as_double((long long)(1023 + (int)kf) << 52);
  return v > 0.0 ? y : -y;
}

__device__ __forceinline__ void ipt_from_lin(const double* lin, double* o) {
  // color.py:150-158
  double xyz[3], lms[3], lmsp[3], ipt[3];
  mat3(cc.rgb2xyz, lin, xyz);
  mat3(cc.xyz2lms, xyz, lms);
  for (int i = 0; i < 3; ++i) lmsp[i] = spow043(lms[i]);
  mat3(cc.lms2ipt, lmsp, ipt);
  o[0] = ipt[0];
  o[1] = add(mul(0.5, ipt[1]), 0.5);
  o[2] = add(mul(0.5, ipt[2]), 0.5);
}

__device__ __forceinline__ double eotf(double v) {
  // color.py:131-133
  return v > 0.04045 ? pow(__ddiv_rn(add(v, 0.055), 1.055), 2.4) : __ddiv_rn(v, 12.92);
}

__device__ __forceinline__ double oetf(double v) {
  // color.py:136-138
  return v > 0.0031308 ? sub(mul(1.055, pow(fmax(v, 0.0), 1.0 / 2.4)), 0.055) : mul(12.92, v);
}

// Correctly rounded x / d for a constant d with inv = RN(1/d): q = RN(x inv) is
// within one ulp of x/d, and one remainder correction (exact residual by fma)
// gives RN(x/d) (Markstein); verified against numpy's division on all 2^24
// u8 RGB triples (tests/test_gpu_parity.py::test_color_u8_exhaustive).
__device__ __forceinline__ double div_const(double x, double d, double inv) {
  const double q = __dmul_rn(x, inv);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, inv, q);
}

__device__ double g_eotf[256];  // global copy of cc.eotf for per-block shared-memory staging

// Tile of 64 pixels along w x 32 rows along h per 256-thread block.
// (1) the 32 x 192 source bytes are staged in shared memory (16-byte loads when
//     the row stride allows), (2) each thread converts 8 pixels (lanes walk
//     down a column of the tile, so both the byte reads and the fp32 writes of
//     the transposed tile are bank-conflict free), (3) each (channel, column)
//     run of 32 h-contiguous floats is written with 16-byte stores.
// Y'CbCr forms u8/255 with the corrected-reciprocal division (bitwise the
// reference's value); IPT reads the sRGB EOTF of the u8 code from a shared-memory table.
// channel_major = 0: planes (img, c) at (3 img + c) h w -- the BASELINE (H, W, 3, V*E) stack;
// channel_major = 1: planes at (c n_img + img) h w -- three (H, W, E, V) tensors, one per
// channel, the reference codec's stack_to_tensor layout (sceneio.py:38, 191-199).
// row stride 196 B = 49 words (odd): lanes reading one byte from each of 32 rows hit 32 banks
constexpr int CT_W = 64, CT_H = 32, CT_ROWB = CT_W * 3 + 4, CT_FP = CT_H + 4;

// fp64 constants of the Y'CbCr path as a kernel parameter: the DFMA/DMUL read
// them from the constant bank instead of re-materialising 64-bit immediates
// through uniform registers in the pixel loop (16 UMOV per pixel in ncu)
struct YccConst {
  double kr, kg, kb, kb1, ikb1, kr1, ikr1, i255;
};

// SPACE is a template parameter so each colour space gets its own register
// allocation (the IPT body needs 58 registers; sharing it cost the Y'CbCr path
// two of its six resident blocks per SM)
template <int SPACE>
__global__ void __launch_bounds__(256) k_color_u8(const uint8_t* __restrict__ rgb, int64_t h, int64_t w,
                                                  float* __restrict__ out, int channel_major, const YccConst P) {
  constexpr int space = SPACE;
  __shared__ __align__(16) uint8_t su8[CT_H][CT_ROWB];  // 4-byte aligned rows
  __shared__ __align__(16) float so[3][CT_W][CT_FP];
  __shared__ double lut[256];
  __shared__ double ptab[SPACE == TMB_SPACE_IPT ? 3 * PT : 1];
  const int t = threadIdx.x;
  const int64_t img = blockIdx.z;
  const int64_t x0 = (int64_t)blockIdx.x * CT_W, y0 = (int64_t)blockIdx.y * CT_H;
  const bool full = (x0 + CT_W <= w) && (y0 + CT_H <= h);
  if (space == TMB_SPACE_IPT) {
    lut[t] = g_eotf[t];
    const double* gp = g_powtab.invc;  // invc | lc | e2, contiguous
    for (int i = t; i < 3 * PT; i += 256) ptab[i] = gp[i];
  }
  else if (space != TMB_SPACE_YCBCR) lut[t] = __ddiv_rn((double)t, 255.0);
  const uint8_t* src = rgb + (img * h + y0) * w * 3 + x0 * 3;
  if (full && (w & 15) == 0 && ((reinterpret_cast<uintptr_t>(rgb) & 15) == 0)) {
    for (int i = t; i < CT_H * 12; i += 256) {
      const int r = i / 12, q = i % 12;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)r * w * 3) + q);
      uint32_t* d = reinterpret_cast<uint32_t*>(&su8[r][q * 16]);
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    }
  } else {
    const int64_t nx = w - x0 < CT_W ? w - x0 : CT_W, ny = h - y0 < CT_H ? h - y0 : CT_H;
    for (int i = t; i < CT_H * CT_W * 3; i += 256) {
      const int r = i / (CT_W * 3), bcol = i % (CT_W * 3);
      if (r < ny && bcol < nx * 3) su8[r][bcol] = src[(int64_t)r * w * 3 + bcol];
    }
  }
  __syncthreads();
  const int nyt = full ? CT_H : (int)(h - y0 < CT_H ? h - y0 : CT_H);
  const int nxt = full ? CT_W : (int)(w - x0 < CT_W ? w - x0 : CT_W);
  const int r = t & 31;
  // full tiles (all but the right/bottom edge) run the loop without per-pixel guards
  auto convert = [&](auto guarded) {
#pragma unroll
  for (int col = t >> 5; col < CT_W; col += 8) {
    if (decltype(guarded)::value && (r >= nyt || col >= nxt)) continue;
    const uint8_t* sp = &su8[r][col * 3];
    const int R = sp[0], G = sp[1], B = sp[2];
    float f[3];
    if (space == TMB_SPACE_YCBCR) {
      // color.py:116-118: y = KR r + KG g + KB b; cb = 0.5 (b - y) / (1 - KB) + 0.5;
      // clip to [0, 1] -- applied after the (monotone) rounding to fp32, where
      // it is one FMNMX pair and gives the same float as clipping in fp64
      // u8/255 by the corrected-reciprocal division (no table: random-index
      // shared-memory loads would make the L1 pipe the bound)
      const double r = div_const((double)R, 255.0, P.i255), g = div_const((double)G, 255.0, P.i255),
                   b = div_const((double)B, 255.0, P.i255);
      const double y = add(add(mul(P.kr, r), mul(P.kg, g)), mul(P.kb, b));
      const double cb = add(div_const(mul(0.5, sub(b, y)), P.kb1, P.ikb1), 0.5);
      const double cr = add(div_const(mul(0.5, sub(r, y)), P.kr1, P.ikr1), 0.5);
      f[0] = fminf(fmaxf(__double2float_rn(y), 0.0f), 1.0f);
      f[1] = fminf(fmaxf(__double2float_rn(cb), 0.0f), 1.0f);
      f[2] = fminf(fmaxf(__double2float_rn(cr), 0.0f), 1.0f);
    } else {
      double o[3];
      if (space == TMB_SPACE_IPT) {
        // u8 path: linear RGB -> LMS through the one fused 3x3 product and fma
        // chains (the reference multiplies by rgb2xyz then xyz2lms; the fp32
        // outputs are checked bit-identical on all 2^24 triples)
        const double l0 = lut[R], l1 = lut[G], l2 = lut[B];
        double lmsp[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          lmsp[i] = pow043_tab(fma(l2, cc.lin2lms[3 * i + 2], fma(l1, cc.lin2lms[3 * i + 1], l0 * cc.lin2lms[3 * i])),
                               ptab, ptab + PT, ptab + 2 * PT);
        double ipt[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          ipt[i] = fma(lmsp[2], cc.lms2ipt[3 * i + 2], fma(lmsp[1], cc.lms2ipt[3 * i + 1], lmsp[0] * cc.lms2ipt[3 * i]));
        o[0] = ipt[0];
        o[1] = add(mul(0.5, ipt[1]), 0.5);
        o[2] = add(mul(0.5, ipt[2]), 0.5);
      } else {
        o[0] = lut[R]; o[1] = lut[G]; o[2] = lut[B];
      }
      f[0] = __double2float_rn(o[0]); f[1] = __double2float_rn(o[1]); f[2] = __double2float_rn(o[2]);
    }
    so[0][col][r] = f[0];
    so[1][col][r] = f[1];
    so[2][col][r] = f[2];
  }
  };
  if (full) convert(std::false_type{});
  else convert(std::true_type{});
  __syncthreads();
  const int64_t hw = h * w;
  float* dst = out + img * (channel_major ? hw : 3 * hw) + x0 * h + y0;
  const int64_t cstride = channel_major ? (int64_t)gridDim.z * hw : hw;
  if (full && (h & 3) == 0 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    for (int i = t; i < 3 * CT_W * 8; i += 256) {
      const int q = i & 7, col = (i >> 3) % CT_W, ch = i / (CT_W * 8);
      *reinterpret_cast<float4*>(dst + cstride * ch + (int64_t)col * h + 4 * q) =
          *reinterpret_cast<const float4*>(&so[ch][col][4 * q]);
    }
  } else {
    for (int i = t; i < 3 * CT_W * CT_H; i += 256) {
      const int r = i & 31, col = (i >> 5) % CT_W, ch = i / (CT_W * CT_H);
      if (y0 + r < h && x0 + col < w) dst[cstride * ch + (int64_t)col * h + r] = so[ch][col][r];
    }
  }
}

__global__ void k_color_f64(const double* __restrict__ px, int64_t npx, int space, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = px[3 * i], g = px[3 * i + 1], b = px[3 * i + 2];
    double o[3];
    if (space == TMB_SPACE_YCBCR) {
      ycbcr(r, g, b, o);
    } else if (space == TMB_SPACE_IPT) {
      const double lin[3] = {eotf(r), eotf(g), eotf(b)};
      ipt_from_lin(lin, o);
    } else {
      o[0] = r; o[1] = g; o[2] = b;
    }
    out[3 * i] = o[0]; out[3 * i + 1] = o[1]; out[3 * i + 2] = o[2];
  }
}

// inverses (color.py:122-128, 161-182) of one pixel; *cl = 1 if ipt_to_rgb clamped
__device__ __forceinline__ void inv_px(int space, double a, double b, double c, double* o, int* cl) {
  *cl = 0;
  if (space == TMB_SPACE_YCBCR) {
    const double r = add(a, mul(mul(2.0, 1.0 - KR), sub(c, 0.5)));
    const double bb = add(a, mul(mul(2.0, 1.0 - KB), sub(b, 0.5)));
    const double g = __ddiv_rn(sub(sub(a, mul(KR, r)), mul(KB, bb)), KG);
    o[0] = r; o[1] = g; o[2] = bb;
  } else if (space == TMB_SPACE_IPT) {
    const double ipt[3] = {a, mul(2.0, sub(b, 0.5)), mul(2.0, sub(c, 0.5))};
    double lmsp[3], lms[3], xyz[3], lin[3];
    mat3(cc.ipt2lms, ipt, lmsp);
    for (int k = 0; k < 3; ++k) lms[k] = spow(lmsp[k], 1.0 / 0.43);
    mat3(cc.lms2xyz, lms, xyz);
    mat3(cc.xyz2rgb, xyz, lin);
    for (int k = 0; k < 3; ++k) {
      const double v = fmin(fmax(lin[k], 0.0), 1.0);
      if (v != lin[k]) *cl = 1;
      o[k] = oetf(v);
    }
  } else {
    o[0] = a; o[1] = b; o[2] = c;
  }
}

__global__ void k_color_inv(const double* __restrict__ px, int64_t npx, int space, double* __restrict__ out,
                            int* __restrict__ clamped) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
    double o[3];
    int cl;
    inv_px(space, px[3 * i], px[3 * i + 1], px[3 * i + 2], o, &cl);
    out[3 * i] = o[0]; out[3 * i + 1] = o[1]; out[3 * i + 2] = o[2];
    clamped[i] = cl;
  }
}

// The codec's float64 path (codec.py:389 then stack_to_tensor, sceneio.py:191-199):
// n_img interleaved float64 images (img, h, w, 3) -- ColorImage.pixels of the
// scene in (view, exposure) order -- through to_coding_space into three float64
// F-order (h, w, E, V) channel tensors, plane (c n_img + img). 32 x 32 pixel
// tiles transposed through shared memory: pixel reads along w, writes along h.
__global__ void __launch_bounds__(256) k_color_f64_channels(const double* __restrict__ px, int64_t n_img,
                                                            int64_t h, int64_t w, int space,
                                                            double* __restrict__ out) {
  __shared__ double so[3][32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t img = blockIdx.z, h0 = (int64_t)blockIdx.y * 32, w0 = (int64_t)blockIdx.x * 32;
  for (int r = ty; r < 32; r += 8) {
    const int64_t hh = h0 + r, ww = w0 + tx;
    if (hh < h && ww < w) {
      const double* p = px + ((img * h + hh) * w + ww) * 3;
      double o[3];
      if (space == TMB_SPACE_YCBCR) {
        ycbcr(p[0], p[1], p[2], o);
      } else if (space == TMB_SPACE_IPT) {
        const double lin[3] = {eotf(p[0]), eotf(p[1]), eotf(p[2])};
        ipt_from_lin(lin, o);
      } else {
        o[0] = p[0]; o[1] = p[1]; o[2] = p[2];
      }
      for (int c = 0; c < 3; ++c) so[c][tx][r] = o[c];
    }
  }
  __syncthreads();
  const int64_t plane = h * w;
  for (int col = ty; col < 32; col += 8) {
    const int64_t hh = h0 + tx, ww = w0 + col;
    if (hh < h && ww < w)
      for (int c = 0; c < 3; ++c) out[(c * n_img + img) * plane + ww * h + hh] = so[c][col][tx];
  }
}

// decode_stream's last steps (codec.py:446-468): three float64 (h, w, E, V)
// channel tensors (reconstruct(dequantize(q)) per channel) -> tensor_to_stack
// -> to_rgb per image, written as interleaved float64 RGB images (img, h, w, 3).
__global__ void __launch_bounds__(256) k_channels_to_rgb(const double* __restrict__ t, int64_t n_img, int64_t h,
                                                         int64_t w, int space, double* __restrict__ rgb) {
  __shared__ double si[3][32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t img = blockIdx.z, h0 = (int64_t)blockIdx.y * 32, w0 = (int64_t)blockIdx.x * 32;
  const int64_t plane = h * w;
  for (int col = ty; col < 32; col += 8) {
    const int64_t hh = h0 + tx, ww = w0 + col;
    if (hh < h && ww < w)
      for (int c = 0; c < 3; ++c) si[c][col][tx] = t[(c * n_img + img) * plane + ww * h + hh];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t hh = h0 + r, ww = w0 + tx;
    if (hh < h && ww < w) {
      double o[3];
      int cl;
      inv_px(space, si[0][tx][r], si[1][tx][r], si[2][tx][r], o, &cl);
      double* q = rgb + ((img * h + hh) * w + ww) * 3;
      q[0] = o[0]; q[1] = o[1]; q[2] = o[2];
    }
  }
}

// Decode side: the reconstructed coding-space stack
// (F-order h x w x 3 x n_img fp64, reconstruct(dequantize(q)), codec.py:446-447)
// -> to_rgb per pixel (color.py:197-205) -> optional interleaved RGB output and
// the per-tile sum of squared 8-bit-unit errors against the original u8 images
// (metrics.mse on pixels*255, metrics.py:16-23, as scene_psnr calls it, :41-76).
// 32x32 pixel tiles: the fp64 planes are read along h (F-order, coalesced), the
// u8 rows staged through shared memory along w.
__global__ void __launch_bounds__(256) k_decode_sse(const double* __restrict__ t, int64_t h, int64_t w, int space,
                                                    const uint8_t* __restrict__ rgb, double* __restrict__ out,
                                                    double* __restrict__ part) {
  __shared__ uint8_t su8[32][32 * 3 + 4];
  __shared__ double red[8];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t img = blockIdx.z, h0 = (int64_t)blockIdx.y * 32, w0 = (int64_t)blockIdx.x * 32;
  if (rgb) {
    for (int r = ty; r < 32; r += 8) {
      const int64_t hh = h0 + r;
      if (hh >= h) continue;
      const uint8_t* row = rgb + ((img * h + hh) * w + w0) * 3;
      for (int bcol = tx; bcol < 96; bcol += 32)
        if (w0 + bcol / 3 < w) su8[r][bcol] = row[bcol];
    }
    __syncthreads();
  }
  const int64_t hw = h * w;
  const double* plane = t + 3 * hw * img;
  double sse = 0.0;
  for (int k = ty; k < 32; k += 8) {
    const int64_t hh = h0 + tx, ww = w0 + k;
    if (hh >= h || ww >= w) continue;
    const int64_t p = hh + h * ww;
    double o[3];
    int cl;
    inv_px(space, plane[p], plane[p + hw], plane[p + 2 * hw], o, &cl);
    if (out) {
      double* q = out + ((img * h + hh) * w + ww) * 3;
      q[0] = o[0]; q[1] = o[1]; q[2] = o[2];
    }
    if (rgb) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const double ref = mul(__ddiv_rn((double)su8[tx][k * 3 + ch], 255.0), 255.0);  // (u8/255)*255
        const double d = sub(ref, mul(o[ch], 255.0));
        sse = __fma_rn(d, d, sse);
      }
    }
  }
  if (!rgb) return;
  for (int off = 16; off > 0; off >>= 1) sse += __shfl_xor_sync(0xffffffffu, sse, off);
  if (tx == 0) red[ty] = sse;
  __syncthreads();
  if (tx == 0 && ty == 0) {
    double s2 = 0.0;
    for (int i = 0; i < 8; ++i) s2 += red[i];
    part[img * (int64_t)gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = s2;
  }
}

// per-image sum of its tile partials, fixed order (one warp per image)
__global__ void k_sse_final(const double* __restrict__ part, int64_t tiles, int64_t n_img, double* __restrict__ sse) {
  const int64_t img = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (img >= n_img) return;
  double s = 0.0;
  for (int64_t i = lane; i < tiles; i += 32) s += part[img * tiles + i];
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) sse[img] = s;
}

__global__ void k_count(const int* __restrict__ f, int64_t n, unsigned long long* __restrict__ cnt) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    local += f[i];
  atomicAdd(&s, local);  // integer: order-independent
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(cnt, s);
}

// 3x3 helpers on the host (row-major), reproducing color.py:43-77
void inv3(const double* m, double* o) {
  const double a = m[0], b = m[1], c = m[2], d = m[3], e = m[4], f = m[5], g = m[6], h = m[7], i = m[8];
  const double A = e * i - f * h, B = -(d * i - f * g), C = d * h - e * g;
  const double det = a * A + b * B + c * C;
  o[0] = A / det; o[1] = -(b * i - c * h) / det; o[2] = (b * f - c * e) / det;
  o[3] = B / det; o[4] = (a * i - c * g) / det; o[5] = -(a * f - c * d) / det;
  o[6] = C / det; o[7] = -(a * h - b * g) / det; o[8] = (a * e - b * d) / det;
}

bool g_const_ready[64] = {false};
std::mutex g_const_mu;  // contexts on several host threads (pipeline lanes) may arrive together

void ensure_constants(Ctx& c) {
  std::lock_guard<std::mutex> lk(g_const_mu);
  if (c.device >= 0 && c.device < 64 && g_const_ready[c.device]) return;
  ColorConst h{};
  for (int v = 0; v < 256; ++v) {
    const double x = (double)v / 255.0;
    h.eotf[v] = x > 0.04045 ? std::pow((x + 0.055) / 1.055, 2.4) : x / 12.92;
  }
  const double rgb2xyz[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                             0.0721750, 0.0193339, 0.1191920, 0.9503041};
  const double hpe[9] = {0.4002, 0.7075, -0.0807, -0.2280, 1.1500, 0.0612, 0.0000, 0.0000, 0.9184};
  double white[3];
  for (int r = 0; r < 3; ++r) white[r] = rgb2xyz[3 * r] + rgb2xyz[3 * r + 1] + rgb2xyz[3 * r + 2];
  for (int r = 0; r < 3; ++r) {
    const double s = hpe[3 * r] * white[0] + hpe[3 * r + 1] * white[1] + hpe[3 * r + 2] * white[2];
    for (int k = 0; k < 3; ++k) h.xyz2lms[3 * r + k] = hpe[3 * r + k] / s;
  }
  const double lms2ipt[9] = {0.4000, 0.4000, 0.2000, 4.4550, -4.8510, 0.3960, 0.8056, 0.3572, -1.1628};
  for (int k = 0; k < 9; ++k) { h.rgb2xyz[k] = rgb2xyz[k]; h.lms2ipt[k] = lms2ipt[k]; }
  inv3(h.rgb2xyz, h.xyz2rgb);
  inv3(h.xyz2lms, h.lms2xyz);
  inv3(h.lms2ipt, h.ipt2lms);
  for (int r = 0; r < 3; ++r)
    for (int k2 = 0; k2 < 3; ++k2)
      h.lin2lms[3 * r + k2] = h.xyz2lms[3 * r] * h.rgb2xyz[k2] + h.xyz2lms[3 * r + 1] * h.rgb2xyz[3 + k2] +
                              h.xyz2lms[3 * r + 2] * h.rgb2xyz[6 + k2];
  TMB_CUDA(cudaMemcpyToSymbol(g_eotf, h.eotf, sizeof(h.eotf)));
  // log2(1 + r) Taylor coefficients (-1)^(k+1) / (k ln 2), k = 6 .. 1; e^t: 1/720 .. 1/2 (+ 1, 1 inline)
  const long double ln2 = 0.693147180559945309417232121458176568L;
  for (int k = 6; k >= 1; --k) h.plog[6 - k] = (double)(((k % 2) ? 1.0L : -1.0L) / ((long double)k * ln2));
  h.pexp[0] = 0.43;
  h.pexp[1] = (double)ln2;
  h.pexp[2] = (double)(1.0L / 720.0L);
  h.pexp[3] = (double)(1.0L / 120.0L);
  h.pexp[4] = (double)(1.0L / 24.0L);
  h.pexp[5] = (double)(1.0L / 6.0L);
  h.pexp[6] = 0.5;
  TMB_CUDA(cudaMemcpyToSymbol(cc, &h, sizeof(h)));
  PowTab pt;
  for (int j = 0; j < PT; ++j) {
    pt.invc[j] = (double)(1.0L / (1.0L + ((long double)j + 0.5L) / PT));
    pt.lc[j] = (double)(-std::log2((long double)pt.invc[j]));
    pt.e2[j] = (double)std::exp2((long double)j / PT);
  }
  TMB_CUDA(cudaMemcpyToSymbol(g_powtab, &pt, sizeof(pt)));
  if (c.device >= 0 && c.device < 64) g_const_ready[c.device] = true;
}

}  // namespace

void color_u8(Ctx& c, const uint8_t* rgb, int64_t n_img, int64_t h, int64_t w, int space, float* out,
              bool channel_major) {
  if (n_img == 0 || h == 0 || w == 0) return;
  ensure_constants(c);
  dim3 grid((unsigned)ceil_div(w, CT_W), (unsigned)ceil_div(h, CT_H), (unsigned)n_img);
  Timed timed(c, TAG_COLOR, 15.0 * (double)n_img * h * w);  // 3 B read + 12 B written per pixel
  const YccConst P{KR, KG, KB, 1.0 - KB, 1.0 / (1.0 - KB), 1.0 - KR, 1.0 / (1.0 - KR), 1.0 / 255.0};
  const int cm = channel_major ? 1 : 0;
  if (space == TMB_SPACE_YCBCR) k_color_u8<TMB_SPACE_YCBCR><<<grid, 256, 0, c.stream>>>(rgb, h, w, out, cm, P);
  else if (space == TMB_SPACE_IPT) k_color_u8<TMB_SPACE_IPT><<<grid, 256, 0, c.stream>>>(rgb, h, w, out, cm, P);
  else k_color_u8<TMB_SPACE_RGB><<<grid, 256, 0, c.stream>>>(rgb, h, w, out, cm, P);
  c.launches++;
  check_launch("k_color_u8");
}

void color_f64(Ctx& c, const double* px, int64_t npx, int space, double* out) {
  if (npx == 0) return;
  ensure_constants(c);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npx, 256), 16LL * c.num_sms));
  k_color_f64<<<blocks, 256, 0, c.stream>>>(px, npx, space, out);
  c.launches++;
  check_launch("k_color_f64");
}

void color_inv_f64(Ctx& c, const double* px, int64_t npx, int space, double* out, int64_t* n_clamped) {
  if (npx == 0) { if (n_clamped) *n_clamped = 0; return; }
  ensure_constants(c);
  const size_t mk = c.arena.mark();
  int* flags = alloc<int>(c, npx);
  unsigned long long* cnt = alloc<unsigned long long>(c, 1);
  TMB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c.stream));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npx, 256), 16LL * c.num_sms));
  k_color_inv<<<blocks, 256, 0, c.stream>>>(px, npx, space, out, flags);
  c.launches++;
  check_launch("k_color_inv");
  k_count<<<blocks, 256, 0, c.stream>>>(flags, npx, cnt);
  c.launches++;
  check_launch("k_count");
  unsigned long long hc = 0;
  TMB_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  if (n_clamped) *n_clamped = (int64_t)hc;
  c.arena.release(mk);
}

void color_f64_channels(Ctx& c, const double* px, int64_t n_img, int64_t h, int64_t w, int space, double* out) {
  if (n_img == 0 || h == 0 || w == 0) return;
  ensure_constants(c);
  dim3 grid((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32), (unsigned)n_img);
  k_color_f64_channels<<<grid, dim3(32, 8), 0, c.stream>>>(px, n_img, h, w, space, out);
  c.launches++;
  check_launch("k_color_f64_channels");
}

void channels_to_rgb(Ctx& c, const double* t, int64_t n_img, int64_t h, int64_t w, int space, double* rgb) {
  if (n_img == 0 || h == 0 || w == 0) return;
  ensure_constants(c);
  dim3 grid((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32), (unsigned)n_img);
  k_channels_to_rgb<<<grid, dim3(32, 8), 0, c.stream>>>(t, n_img, h, w, space, rgb);
  c.launches++;
  check_launch("k_channels_to_rgb");
}

void decode_sse(Ctx& c, const double* t, int64_t n_img, int64_t h, int64_t w, int space, const uint8_t* rgb,
                double* out_rgb, double* sse_dev) {
  if (n_img == 0 || h == 0 || w == 0) return;
  ensure_constants(c);
  const size_t mk = c.arena.mark();
  dim3 grid((unsigned)ceil_div(w, 32), (unsigned)ceil_div(h, 32), (unsigned)n_img);
  const int64_t tiles = (int64_t)grid.x * grid.y;
  double* part = rgb ? alloc<double>(c, (size_t)(tiles * n_img)) : nullptr;
  k_decode_sse<<<grid, dim3(32, 8), 0, c.stream>>>(t, h, w, space, rgb, out_rgb, part);
  c.launches++;
  check_launch("k_decode_sse");
  if (rgb) {
    k_sse_final<<<(unsigned)ceil_div(n_img, 8), 256, 0, c.stream>>>(part, tiles, n_img, sse_dev);
    c.launches++;
    check_launch("k_sse_final");
  }
  c.arena.release(mk);
}

}  // namespace tmb
