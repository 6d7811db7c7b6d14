// Research microbenchmark: cost of one grid-wide barrier on B200 with one
// 512-thread block per SM (the k_sytrd_smem configuration), each block having
// just stored a few values to global memory (the p_{k+1} publication).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
// Variants: 0 cg::grid.sync; 1 fence + atomicAdd + acquire poll; 2 red.release +
// acquire poll (no separate fence); 3 cluster-of-2 hierarchy (barrier.cluster,
// one leader per pair does 2).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__global__ void __launch_bounds__(512, 1) k_bar(unsigned* cnt, double* sink, int iters, long long* out) {
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const unsigned nb = gridDim.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (tid < 16) sink[(blockIdx.x * 16 + tid) + (size_t)(it & 7) * gridDim.x * 16] = it;  // the p publication
    if constexpr (V == 0) {
      grid.sync();
    } else if constexpr (V == 1) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        const unsigned target = nb * (unsigned)(it + 1);
        while (ld_acquire(cnt) < target) {
        }
      }
      __syncthreads();
    } else if constexpr (V == 2) {
      __syncthreads();
      if (tid == 0) {
        red_release(cnt, 1u);
        const unsigned target = nb * (unsigned)(it + 1);
        while (ld_acquire(cnt) < target) {
        }
      }
      __syncthreads();
    } else if constexpr (V == 4) {
      // per-block arrival flags (32 words apart); every block polls all of them
      __syncthreads();
      if (tid == 0) st_release(cnt + 32 * (blockIdx.x + 1), (unsigned)(it + 1));
      if (tid < (int)nb)
        while (ld_acquire(cnt + 32 * (tid + 1)) < (unsigned)(it + 1)) {
        }
      __syncthreads();
    } else if constexpr (V == 5) {
      // per-block arrival flags; block 0 gathers them and releases everyone with one flag
      __syncthreads();
      if (tid == 0) st_release(cnt + 32 * (blockIdx.x + 1), (unsigned)(it + 1));
      if (blockIdx.x == 0) {
        if (tid < (int)nb)
          while (ld_acquire(cnt + 32 * (tid + 1)) < (unsigned)(it + 1)) {
          }
        __syncthreads();
        if (tid == 0) st_release(cnt, (unsigned)(it + 1));
      } else if (tid == 0) {
        while (ld_acquire(cnt) < (unsigned)(it + 1)) {
        }
      }
      __syncthreads();
    } else {
      // cluster of 2: both CTAs arrive at the cluster barrier, rank 0 publishes
      // the pair's arrival and polls, then releases its partner
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      unsigned rank;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
      if (rank == 0 && tid == 0) {
        red_release(cnt, 1u);
        const unsigned target = (nb / 2) * (unsigned)(it + 1);
        while (ld_acquire(cnt) < target) {
        }
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

template <int V>
void run(int nsm, int iters, bool cluster) {
  unsigned* cnt;
  double* sink;
  long long* out;
  cudaMalloc(&cnt, 4 * 32 * 160);
  cudaMemset(cnt, 0, 4 * 32 * 160);
  cudaMalloc(&sink, sizeof(double) * nsm * 16 * 8);
  cudaMalloc(&out, sizeof(long long) * nsm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 0;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeCooperative;
  attr[na].val.cooperative = 1;
  ++na;
  if (cluster) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar<V>, cnt, sink, 10, out);  // warm-up
  cudaDeviceSynchronize();
  cudaMemset(cnt, 0, 4 * 32 * 160);
  cudaEventRecord(a);
  e = cudaLaunchKernelEx(&cfg, k_bar<V>, cnt, sink, iters, out);
  cudaEventRecord(b);
  cudaError_t e2 = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long h[1024];
  cudaMemcpy(h, out, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  long long mx = 0, mn = 1ll << 60;
  for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
  std::printf("variant %d%s: %s/%s  %.3f us/barrier (events), clock64 cycles/barrier min %lld max %lld\n", V,
              cluster ? " (cluster 2)" : "", cudaGetErrorString(e), cudaGetErrorString(e2), 1e3 * ms / iters, mn, mx);
  cudaFree(cnt);
  cudaFree(sink);
  cudaFree(out);
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = argc > 1 ? std::atoi(argv[1]) : 20000;
  run<0>(nsm, iters, false);
  run<1>(nsm, iters, false);
  run<2>(nsm, iters, false);
  run<3>(nsm, iters, true);
  run<4>(nsm, iters, false);
  run<5>(nsm, iters, false);
  run<0>(nsm, iters, false);
  return 0;
}
