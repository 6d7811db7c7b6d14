// Latent-block byte format on the device: the quantised
// core levels of the reference's latent path are stored as zigzag-mapped
// LEB128 varints in F order (codec.py:285-291 -> entropy.encode_ints,
// entropy.py:55-111) and read back by decode_ints (entropy.py:88-117).
//
// Encode: per-value byte length -> block sums -> one-block scan of the block
// sums -> per-block local scan + byte scatter. Decode: terminator flags (byte
// < 0x80) -> the same two-level scan gives each terminator its value index ->
// each value gathers its <= 10 bytes. Byte traffic is coalesced in both
// directions; everything is integer work (HBM/latency-bound, no tensor cores).
#include "tmb_internal.cuh"

namespace tmb {
namespace {

constexpr int LT = 1024;        // elements per block (one per thread)
constexpr int MAX_VARINT = 10;  // 64 bits / 7, entropy.py:34

__device__ __forceinline__ uint64_t zigzag(int64_t v) {
  return (static_cast<uint64_t>(v) << 1) ^ static_cast<uint64_t>(v >> 63);  // entropy.py:55-58
}

__device__ __forceinline__ int varint_len(uint64_t u) {
  int n = 1;
  while (u >= 0x80) { u >>= 7; ++n; }
  return n;
}

// exclusive block scan of one int64 per thread (blockDim == LT); returns the block total
__device__ __forceinline__ int64_t block_exscan(int64_t v, int64_t* sh, int64_t* excl) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = sh[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  *excl = x - v + (w > 0 ? sh[w - 1] : 0);
  const int64_t total = sh[31];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(LT) k_enc_sums(const int64_t* __restrict__ lv, int64_t n, int64_t* __restrict__ bsum) {
  __shared__ int64_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x;
  const int64_t len = i < n ? varint_len(zigzag(lv[i])) : 0;
  int64_t ex;
  const int64_t tot = block_exscan(len, sh, &ex);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of nb block totals in place, one block; off[nb] = grand total
__global__ void __launch_bounds__(LT) k_scan_blocks(int64_t* __restrict__ off, int64_t nb) {
  __shared__ int64_t sh[32];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += LT) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? off[i] : 0;
    int64_t ex;
    const int64_t tot = block_exscan(v, sh, &ex);
    if (i < nb) off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) off[nb] = carry;
}

__global__ void __launch_bounds__(LT) k_enc_write(const int64_t* __restrict__ lv, int64_t n,
                                                  const int64_t* __restrict__ boff, uint8_t* __restrict__ out,
                                                  int64_t cap) {
  __shared__ int64_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x;
  uint64_t u = i < n ? zigzag(lv[i]) : 0;
  const int len = i < n ? varint_len(u) : 0;
  int64_t ex;
  block_exscan(len, sh, &ex);
  const int64_t pos = boff[blockIdx.x] + ex;
  if (i < n && pos + len <= cap) {
    for (int j = 0; j < len; ++j) {  // low group first, continuation bit on all but the last
      const uint8_t b = static_cast<uint8_t>(u & 0x7F) | (j + 1 < len ? 0x80 : 0);
      out[pos + j] = b;
      u >>= 7;
    }
  }
}

// decode pass 1: terminators per block
__global__ void __launch_bounds__(LT) k_dec_sums(const uint8_t* __restrict__ in, int64_t nbytes,
                                                 int64_t* __restrict__ bsum) {
  __shared__ int64_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x;
  const int64_t t = (i < nbytes && in[i] < 0x80) ? 1 : 0;
  int64_t ex;
  const int64_t tot = block_exscan(t, sh, &ex);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// decode pass 2: terminator at byte i with value index j records ends[j] = i
__global__ void __launch_bounds__(LT) k_dec_ends(const uint8_t* __restrict__ in, int64_t nbytes, int64_t count,
                                                 const int64_t* __restrict__ boff, int64_t* __restrict__ ends) {
  __shared__ int64_t sh[32];
  const int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x;
  const int64_t t = (i < nbytes && in[i] < 0x80) ? 1 : 0;
  int64_t ex;
  block_exscan(t, sh, &ex);
  const int64_t j = boff[blockIdx.x] + ex;
  if (t && j < count) ends[j] = i;
}

// decode pass 3: value j spans (ends[j-1], ends[j]]; flag[0] |= 1 when a value exceeds 10 bytes
__global__ void k_dec_values(const uint8_t* __restrict__ in, const int64_t* __restrict__ ends, int64_t count,
                             int64_t* __restrict__ lv, int* __restrict__ flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t start = j == 0 ? 0 : ends[j - 1] + 1, end = ends[j];
    const int64_t len = end - start + 1;
    if (len > MAX_VARINT) { atomicOr(flag, 1); lv[j] = 0; continue; }
    uint64_t u = 0;
    for (int64_t q = 0; q < len; ++q) u |= static_cast<uint64_t>(in[start + q] & 0x7F) << (7 * q);
    lv[j] = static_cast<int64_t>(u >> 1) ^ -static_cast<int64_t>(u & 1);  // entropy.py:61-63
  }
}

}  // namespace

int64_t varint_encode(Ctx& c, const int64_t* levels, int64_t n, uint8_t* out, int64_t cap) {
  if (n <= 0) return 0;
  const size_t mk = c.arena.mark();
  const int64_t nb = ceil_div(n, LT);
  int64_t* off = alloc<int64_t>(c, (size_t)nb + 1);
  k_enc_sums<<<(unsigned)nb, LT, 0, c.stream>>>(levels, n, off);
  c.launches++;
  check_launch("k_enc_sums");
  k_scan_blocks<<<1, LT, 0, c.stream>>>(off, nb);
  c.launches++;
  check_launch("k_scan_blocks");
  int64_t total = 0;
  TMB_CUDA(cudaMemcpyAsync(&total, off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  if (total > cap) {
    c.arena.release(mk);
    throw Error(TMB_EINVAL, "varint output buffer too small: need " + std::to_string(total) + " bytes");
  }
  k_enc_write<<<(unsigned)nb, LT, 0, c.stream>>>(levels, n, off, out, cap);
  c.launches++;
  check_launch("k_enc_write");
  c.arena.release(mk);
  return total;
}

int64_t varint_decode(Ctx& c, const uint8_t* in, int64_t nbytes, int64_t count, int64_t* levels) {
  if (count <= 0) return 0;
  if (nbytes <= 0) throw Error(TMB_EINVAL, "varint stream truncated: 0 values, expected " + std::to_string(count));
  const size_t mk = c.arena.mark();
  const int64_t nb = ceil_div(nbytes, LT);
  int64_t* off = alloc<int64_t>(c, (size_t)nb + 1);
  int64_t* ends = alloc<int64_t>(c, (size_t)count);
  int* flag = alloc<int>(c, 1);
  TMB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
  k_dec_sums<<<(unsigned)nb, LT, 0, c.stream>>>(in, nbytes, off);
  c.launches++;
  check_launch("k_dec_sums");
  k_scan_blocks<<<1, LT, 0, c.stream>>>(off, nb);
  c.launches++;
  check_launch("k_scan_blocks");
  k_dec_ends<<<(unsigned)nb, LT, 0, c.stream>>>(in, nbytes, count, off, ends);
  c.launches++;
  check_launch("k_dec_ends");
  int64_t found = 0;
  TMB_CUDA(cudaMemcpyAsync(&found, off + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  if (found < count) {
    c.arena.release(mk);
    throw Error(TMB_EINVAL, "varint stream truncated: " + std::to_string(found) + " values, expected " +
                                std::to_string(count));
  }
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 16LL * c.num_sms));
  k_dec_values<<<blocks, 256, 0, c.stream>>>(in, ends, count, levels, flag);
  c.launches++;
  check_launch("k_dec_values");
  int hflag = 0;
  int64_t last = 0;
  TMB_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaMemcpyAsync(&last, ends + count - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  TMB_CUDA(cudaStreamSynchronize(c.stream));
  c.arena.release(mk);
  if (hflag) throw Error(TMB_EINVAL, "varint longer than 10 bytes");
  return last + 1;
}

}  // namespace tmb
