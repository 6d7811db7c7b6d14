// Microbenchmarks for design decisions: FP64 DMMA vs DFMA throughput, grid-sync latency.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_dmma(double* out, int iters) {
  double a[4], b[2], c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = 0.5 + i * 1e-3;
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0; for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma16(double* out, int iters) {
  double a[8], b[4], c[4][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i * 1e-3;
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double x[8], y = 1.0000001 + threadIdx.x * 1e-9, z = 1e-9;
  for (int i = 0; i < 8; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float x[8], y = 1.0000001f + threadIdx.x * 1e-9f, z = 1e-9f;
  for (int i = 0; i < 8; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], y, z);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0f) out[0] = s;
}

__global__ void k_gridsync(int n, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = n;
}

int main() {
  double* d; cudaMalloc(&d, 64); int* di; cudaMalloc(&di, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float ms;
  for (int wpb : {4, 8, 16}) {
    int iters = 4096; int blocks = sms * 2; int thr = 32 * wpb;
    k_dmma<<<blocks, thr>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma<<<blocks, thr>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * (double)blocks * wpb;
    printf("dmma m16n8k8 warps/blk=%d: %.1f TFLOP/s\n", wpb, fl / ms / 1e9);
    k_dmma16<<<blocks, thr>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma16<<<blocks, thr>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4.0 * iters * (double)blocks * wpb;
    printf("dmma m16n8k16 warps/blk=%d: %.1f TFLOP/s\n", wpb, fl / ms / 1e9);
    k_dfma<<<blocks, thr>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<<<blocks, thr>>>(d, iters * 8); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * iters * 8.0 * blocks * thr;
    printf("dfma warps/blk=%d: %.1f TFLOP/s\n", wpb, fl / ms / 1e9);
    k_ffma<<<blocks, thr>>>((float*)d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_ffma<<<blocks, thr>>>((float*)d, iters * 8); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ffma warps/blk=%d: %.1f TFLOP/s\n", wpb, fl / ms / 1e9);
  }
  for (int thr : {256, 512}) {
    int n = 20000; void* args[] = {&n, &di};
    cudaLaunchCooperativeKernel((void*)k_gridsync, sms, thr, args, 0, 0); cudaDeviceSynchronize();
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_gridsync, sms, thr, args, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync %d blocks x %d thr: %.3f us/sync (err=%s)\n", sms, thr, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
