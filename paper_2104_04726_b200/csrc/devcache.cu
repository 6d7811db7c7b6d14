// Per-device caches of kernel attributes and occupancy. cudaFuncSetAttribute
// and the occupancy calculator act per device context, so a cache keyed only
// by kernel (a function-level static) is wrong for a second device in the same
// process and racy for two host threads; these are keyed by (device, kernel,
// shape) and guarded by one mutex (lookups cost ~100 ns against ~us launches).
#include <map>
#include <mutex>
#include <tuple>

#include "tmb_internal.cuh"

namespace tmb {
namespace {
std::mutex g_mu;
std::map<std::pair<int, const void*>, size_t> g_smem;                      // max dynamic smem set so far
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;           // blocks per SM
}  // namespace

void set_smem_attr(Ctx& c, const void* fn, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  size_t& cur = g_smem[{c.device, fn}];
  if (cur >= bytes) return;
  TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

int blocks_per_sm(Ctx& c, const void* fn, int threads, size_t smem) {
  std::lock_guard<std::mutex> lk(g_mu);
  const auto key = std::make_tuple(c.device, fn, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per_sm = 0;
  TMB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  g_occ[key] = per_sm;
  return per_sm;
}

}  // namespace tmb
