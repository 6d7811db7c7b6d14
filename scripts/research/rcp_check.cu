// Accuracy of the MUFU fp64 reciprocal seed and of two refinements, against
// the correctly rounded 1/b (__drcp_rn): two Newton steps (4 dependent DFMA)
// vs the cubic correction r0 (1 + e + e^2) (3 dependent DFMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 rcp_check.cu -o rcp_check && ./rcp_check
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ double seed(double b) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b)); return r; }
__device__ double newton2(double b) {
  double r = seed(b);
  double e = fma(-b, r, 1.0); r = fma(r, e, r);
  e = fma(-b, r, 1.0); return fma(r, e, r);
}
__device__ double cubic(double b) {
  const double r = seed(b);
  const double e = fma(-b, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ unsigned long long ulps(double a, double b) {
  long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return (unsigned long long)(x > y ? x - y : y - x);
}
__global__ void k(unsigned long long* out, double* rel) {
  unsigned long long s = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned long long m0 = 0, m1 = 0, m2 = 0; double e0 = 0;
  for (int it = 0; it < 4096; ++it) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double mant = 1.0 + (double)(s >> 12) * 0x1p-52;
    const int ex = (int)((s >> 3) % 200) - 100;
    const double b = ((s & 1) ? -1.0 : 1.0) * ldexp(mant, ex);
    const double ref = __drcp_rn(b);
    e0 = fmax(e0, fabs(seed(b) * b - 1.0));
    unsigned long long u1 = ulps(newton2(b), ref), u2 = ulps(cubic(b), ref);
    m1 = u1 > m1 ? u1 : m1; m2 = u2 > m2 ? u2 : m2;
  }
  atomicMax(out + 1, m1); atomicMax(out + 2, m2);
  atomicMax(out + 0, (unsigned long long)__double_as_longlong(e0));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
  k<<<1024, 256>>>(d, nullptr);
  unsigned long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  double e0; memcpy(&e0, &h[0], 8);
  printf("seed max rel err %.3e (2^%.1f); newton2 max ulps %llu; cubic max ulps %llu (1G samples)\n", e0, log2(e0), h[1], h[2]);
  return 0;
}
