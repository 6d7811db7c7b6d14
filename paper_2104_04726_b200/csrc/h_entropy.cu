// Host-side entropy stage of the latent stream (entropy.py:37-52 tag 1 with the
// coder of _kernels_py.py:24-109 / _kernels.pyx:27-141). This is serial byte
// work after the device path, kept native so the drop-in
// encode_stream / decode_stream (codec.py:377-468) produce and read streams in
// the reference's exact format.
//
// The coder: carryless 32-bit range coder (Subbotin) over an order-0 adaptive
// model of 256 byte counts, each starting at 1, +32 per coded symbol, all
// counts halved rounding up when the total reaches 2^16. The reference finds
// cumulative counts by a linear scan; here a Fenwick tree gives the same
// integers in 8 steps (prefix sums for the encoder, a descent for the
// decoder's symbol search), so the bytes are identical.
#include <cstdint>
#include <cstring>

#include "tmb.h"

namespace {

constexpr int64_t kTop = int64_t(1) << 24, kBot = int64_t(1) << 16, kMask = 0xFFFFFFFFLL;
constexpr int kSyms = 256, kInc = 32;
constexpr int64_t kMaxTotal = int64_t(1) << 16;

struct Model {
  int64_t cnt[kSyms];
  int64_t tree[kSyms + 1];  // Fenwick tree over cnt, 1-based
  int64_t total;

  Model() {
    for (int i = 0; i < kSyms; ++i) cnt[i] = 1;
    rebuild();
  }
  void rebuild() {
    total = 0;
    for (int i = 0; i <= kSyms; ++i) tree[i] = 0;
    for (int i = 0; i < kSyms; ++i) {
      total += cnt[i];
      for (int j = i + 1; j <= kSyms; j += j & -j) tree[j] += cnt[i];
    }
  }
  int64_t prefix(int s) const {  // cnt[0] + ... + cnt[s-1]
    int64_t acc = 0;
    for (int j = s; j > 0; j -= j & -j) acc += tree[j];
    return acc;
  }
  // smallest s with prefix(s + 1) > v (v < total); *cum = prefix(s)
  int find(int64_t v, int64_t* cum) const {
    if (v < 0) { *cum = 0; return 0; }
    int pos = 0;
    int64_t acc = 0;
    for (int step = kSyms; step > 0; step >>= 1) {
      const int nx = pos + step;
      if (nx <= kSyms && acc + tree[nx] <= v) { pos = nx; acc += tree[nx]; }
    }
    *cum = acc;
    return pos;  // 0-based symbol index
  }
  void update(int s) {
    cnt[s] += kInc;
    for (int j = s + 1; j <= kSyms; j += j & -j) tree[j] += kInc;
    total += kInc;
    if (total >= kMaxTotal) {
      for (int i = 0; i < kSyms; ++i) cnt[i] = (cnt[i] + 1) >> 1;
      rebuild();
    }
  }
};

inline int64_t floordiv(int64_t a, int64_t b) {  // Python's // for b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

}  // namespace

extern "C" {

int tmb_rc_bound(int64_t n, int64_t* cap) {
  if (n < 0 || !cap) return TMB_EINVAL;
  // a symbol narrows the range by at most total/count < 2^16 and renormalisation
  // restores at least 2^16, so a few bytes per symbol at most; 4n + 16 is loose
  *cap = 4 * n + 16;
  return TMB_OK;
}

int tmb_rc_encode(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap, int64_t* n_out) {
  if (n < 0 || (n > 0 && !in) || !out || !n_out) return TMB_EINVAL;
  Model m;
  int64_t low = 0, rng = kMask, pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int s = in[i];
    const int64_t cum = m.prefix(s);
    rng /= m.total;
    low += cum * rng;
    rng *= m.cnt[s];
    for (;;) {
      if ((low ^ (low + rng)) < kTop) {
      } else if (rng < kBot) {
        rng = (-low) & (kBot - 1);
      } else {
        break;
      }
      if (pos >= cap) return TMB_EINVAL;
      out[pos++] = (uint8_t)((low >> 24) & 0xFF);
      rng = (rng << 8) & kMask;
      low = (low << 8) & kMask;
    }
    m.update(s);
  }
  for (int k = 0; k < 4; ++k) {
    if (pos >= cap) return TMB_EINVAL;
    out[pos++] = (uint8_t)((low >> 24) & 0xFF);
    low = (low << 8) & kMask;
  }
  *n_out = pos;
  return TMB_OK;
}

int tmb_rc_decode(const uint8_t* in, int64_t n_in, int64_t n, uint8_t* out) {
  if (n_in < 0 || n < 0 || (n_in > 0 && !in) || (n > 0 && !out)) return TMB_EINVAL;
  Model m;
  int64_t low = 0, rng = kMask, code = 0, pos = 0;
  auto next = [&]() -> int64_t { const int64_t b = pos < n_in ? in[pos] : 0; ++pos; return b; };
  for (int k = 0; k < 4; ++k) code = ((code << 8) | next()) & kMask;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = rng / m.total;
    int64_t v = floordiv(code - low, r);
    if (v >= m.total) v = m.total - 1;
    int64_t cum;
    const int s = m.find(v, &cum);
    low += cum * r;
    rng = r * m.cnt[s];
    for (;;) {
      if ((low ^ (low + rng)) < kTop) {
      } else if (rng < kBot) {
        rng = (-low) & (kBot - 1);
      } else {
        break;
      }
      code = ((code << 8) | next()) & kMask;
      rng = (rng << 8) & kMask;
      low = (low << 8) & kMask;
    }
    out[i] = (uint8_t)s;
    m.update(s);
  }
  return TMB_OK;
}

}  // extern "C"
