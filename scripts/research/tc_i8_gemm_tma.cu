// Research prototype (not part of libtmb), step 2: tcgen05 kind::i8 GEMM with
// TMA staging (SWIZZLE_128B tiles, the canonical UMMA K-major SW128 layout),
// a 4-deep full/empty mbarrier ring and warp specialisation:
//   warp 0 (one lane): TMA producer      warp 1 (one lane): MMA issuer
//   warps 0..3 after the main loop: TMEM -> registers -> global epilogue.
// C[M,N] int32 = A[M,K] int8 (K-major) * B[N,K]^T int8 (K-major).
// Bounded mbarrier waits trap instead of hanging.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8_gemm_tma tc_i8_gemm_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>

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

constexpr int BM = 128, BN = 256, BK = 128, ST = 4, NTH = 128;
constexpr uint32_t A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major), 16 B
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // version 1
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (long long it = 0; it < 400000000LL; ++it) {
    uint32_t done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
  }
  asm volatile("trap;");
}

__global__ void __launch_bounds__(NTH, 1) k_i8gemm_tma(const __grid_constant__ CUtensorMap ta,
                                                       const __grid_constant__ CUtensorMap tb,
                                                       int32_t* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[ST], empty[ST], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = K / BK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % ST;
      if (kt >= ST) mbar_wait(saddr(&empty[st]), ((kt / ST) - 1) & 1);
      const uint32_t fb = saddr(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE_BYTES) : "memory");
      const uint32_t da = saddr(sm + st * STAGE_BYTES), db = da + A_BYTES;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(da), "l"(&ta), "r"(kt * BK), "r"(m0), "r"(fb) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(db), "l"(&tb), "r"(kt * BK), "r"(n0), "r"(fb) : "memory");
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % ST;
      mbar_wait(saddr(&full[st]), (kt / ST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = saddr(sm + st * STAGE_BYTES), b0 = a0 + A_BYTES;
#pragma unroll
      for (int s = 0; s < BK / 32; ++s) {
        const uint64_t ad = sdesc_sw128(a0 + s * 32), bd = sdesc_sw128(b0 + s * 32);
        const uint32_t acc = (kt > 0 || s > 0) ? 1u : 0u;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&empty[st])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&done)));
  }
  __syncwarp();
  mbar_wait(saddr(&done), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < BN; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int4* dst = reinterpret_cast<int4*>(C + (size_t)(m0 + warp * 32 + lane) * N + n0 + c0);
    dst[0] = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
    dst[1] = make_int4((int)v[4], (int)v[5], (int)v[6], (int)v[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeFn enc, void* base, uint64_t rows, uint64_t kbytes, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {kbytes, rows};
  const cuuint64_t strides[1] = {kbytes};
  const cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { std::fprintf(stderr, "cuTensorMapEncodeTiled failed %d\n", (int)r); std::exit(1); }
  return m;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? std::atoi(argv[1]) : 256, N = argc > 2 ? std::atoi(argv[2]) : 256,
            K = argc > 3 ? std::atoi(argv[3]) : 256, reps = argc > 4 ? std::atoi(argv[4]) : 5;
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
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  const CUtensorMap ta = make_map((EncodeFn)fn, dA, M, K, BM), tb = make_map((EncodeFn)fn, dB, N, K, BN);
  const size_t smem = (size_t)ST * STAGE_BYTES + 1024;
  CK(cudaFuncSetAttribute(k_i8gemm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  k_i8gemm_tma<<<grid, NTH, smem>>>(ta, tb, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> hC((size_t)M * N);
  CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
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
    k_i8gemm_tma<<<grid, NTH, smem>>>(ta, tb, dC, M, N, K);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  std::printf("M=%d N=%d K=%d: %.3f ms, %.1f TOPS\n", M, N, K, best, 2.0 * M * N * (double)K / best / 1e9);
  return bad ? 1 : 0;
}
