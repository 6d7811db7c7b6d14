// Research prototype (not part of libtmb): a minimal tcgen05 kind::i8 GEMM,
// C[M,N] (int32) = A[M,K] (int8, K-major) * B[N,K]^T (int8, K-major), to
// measure whether an Ozaki-style int8 split of the fp64 TTM/Gram contractions
// can beat the DMMA pipe on this B200.
//
// One CTA per 128 x BN output tile, 128 threads: all threads stage A/B K-chunks
// (128 B of K) with cp.async into the canonical no-swizzle K-major UMMA layout
// (8-row x 16-byte core matrices), one thread issues tcgen05.mma (K = 32 B per
// instruction) into a TMEM accumulator and commits to a per-stage mbarrier;
// the epilogue reads TMEM with tcgen05.ld.32x32b. Every mbarrier wait is
// bounded (trap on timeout) so a descriptor mistake cannot hang the GPU.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8_gemm tc_i8_gemm.cu
// Run:   ./tc_i8_gemm M N K [reps]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

constexpr int BM = 128, BK = 128, ST = 3, NTH = 128;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (long long it = 0; it < 200000000LL; ++it) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
  }
  asm volatile("trap;");
}

template <int BN>
__global__ void __launch_bounds__(NTH, 1) k_i8gemm(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                   int32_t* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                                 // ST x (BM x BK)
  uint8_t* sB = sm + ST * BM * BK;                  // ST x (BN x BK)
  __shared__ __align__(8) uint64_t bar[ST];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  // canonical K-major no-swizzle tile: core matrix (8 rows x 16 B) = 128 B;
  // core (rg, kg) at (rg * (BK/16) + kg) * 128  -> LBO (along K) 128 B, SBO (along rows) (BK/16)*128 B
  constexpr uint32_t LBO = 128, SBO = (BK / 16) * 128;
  auto load = [&](int st, int kt) {
    const int k0 = kt * BK;
    uint8_t* dA = sA + st * BM * BK;
    uint8_t* dB = sB + st * BN * BK;
    for (int c = tid; c < BM * (BK / 16); c += NTH) {
      const int r = c / (BK / 16), kg = c % (BK / 16);
      const uint32_t dst = saddr(dA + ((r / 8) * (BK / 16) + kg) * 128 + (r % 8) * 16);
      const int8_t* src = A + (size_t)(m0 + r) * K + k0 + kg * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
    for (int c = tid; c < BN * (BK / 16); c += NTH) {
      const int r = c / (BK / 16), kg = c % (BK / 16);
      const uint32_t dst = saddr(dB + ((r / 8) * (BK / 16) + kg) * 128 + (r % 8) * 16);
      const int8_t* src = B + (size_t)(n0 + r) * K + k0 + kg * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
  };
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  const int KT = K / BK;
  uint32_t uses[ST] = {0, 0, 0};
  for (int s = 0; s < ST - 1 && s < KT; ++s) {
    load(s, s);
    asm volatile("cp.async.commit_group;");
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % ST;
    // refill the stage the MMAs of iteration kt-1 are reading only after they completed
    const int nk = kt + ST - 1;
    if (nk < KT) {
      const int ns = nk % ST;
      if (nk >= ST) mbar_wait(saddr(&bar[ns]), (uses[ns] - 1) & 1);
      load(ns, nk);
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 1));
    asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes -> visible to the tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = saddr(sA + st * BM * BK), b0 = saddr(sB + st * BN * BK);
#pragma unroll
      for (int s = 0; s < BK / 32; ++s) {
        const uint64_t ad = sdesc(a0 + s * 2 * 128, LBO, SBO), bd = sdesc(b0 + s * 2 * 128, LBO, SBO);
        const uint32_t acc = (kt > 0 || s > 0) ? 1u : 0u;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar[st])));
    }
    uses[st]++;
  }
  // all MMAs done when the last commit's barrier phase completes
  const int last = (KT - 1) % ST;
  mbar_wait(saddr(&bar[last]), (uses[last] - 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w owns TMEM lanes 32w..32w+31 (= rows), 8 columns per load
  for (int c0 = 0; c0 < BN; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int32_t* dst = C + (size_t)(m0 + warp * 32 + lane) * N + n0 + c0;
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? std::atoi(argv[1]) : 256, N = argc > 2 ? std::atoi(argv[2]) : 256,
            K = argc > 3 ? std::atoi(argv[3]) : 256, reps = argc > 4 ? std::atoi(argv[4]) : 5;
  constexpr int BN = 256;
  if (M % BM || N % BN || K % BK) { std::fprintf(stderr, "M%%128, N%%256, K%%128 required\n"); return 2; }
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int8_t)((s >> 24) & 0xFF); };
  for (auto& x : hA) x = rnd();
  for (auto& x : hB) x = rnd();
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dC, sizeof(int32_t) * (size_t)M * N));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  const size_t smem = (size_t)ST * (BM * BK + BN * BK);
  CK(cudaFuncSetAttribute(k_i8gemm<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  k_i8gemm<BN><<<grid, NTH, smem>>>(dA, dB, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> hC((size_t)M * N);
  CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
  // verify a sample of entries
  long long bad = 0, checked = 0;
  for (int i = 0; i < M; i += (M > 512 ? 37 : 1))
    for (int j = 0; j < N; j += (N > 512 ? 41 : 1)) {
      long long ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)hA[(size_t)i * K + k] * (int)hB[(size_t)j * K + k];
      if (ref != hC[(size_t)i * N + j]) {
        if (bad < 5) std::printf("mismatch C[%d,%d] = %d, ref %lld\n", i, j, hC[(size_t)i * N + j], ref);
        ++bad;
      }
      ++checked;
    }
  std::printf("verify: %lld / %lld mismatches\n", bad, checked);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    k_i8gemm<BN><<<grid, NTH, smem>>>(dA, dB, dC, M, N, K);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  std::printf("M=%d N=%d K=%d: %.3f ms, %.1f TOPS\n", M, N, K, best, 2.0 * M * N * (double)K / best / 1e9);
  return bad ? 1 : 0;
}
