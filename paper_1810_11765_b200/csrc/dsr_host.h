// dsr_host.h -- host-side plumbing shared by the C ABI and the app tables.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include "dsr_device.cuh"
#include "dsr_doall.cuh"

namespace dsr {

struct LaunchCtx {
  DevHeap h;
  cudaStream_t st;
  int grid;            // persistent grid size for element loops (multiple of #SMs)
  int sms;
  int rk = -1;         // do-all body: range of R (-1 = all; k = k-th type of a subtree do-all)
};

struct MethodInfo {
  // 1: the method may allocate or destroy objects, so the pass needs the
  // iteration-bitmap snapshot.  Without it a visitor could see slots
  // allocated during the pass, or -- when a block empties and is invalidated
  // (all bits set, Alg. 9) -- phantom objects in slots that were already dead.
  // 2: snapshot + dynamic work distribution (k_doall), for passes whose
  // per-object cost is very uneven (several allocations per visit).
  // 3: snapshot + blocked distribution (one contiguous range of R per warp),
  // for passes that free whole blocks.
  // 4: the method enumerates its objects through an app index (GoL's cell
  // grid): no prologue, no block list.
  int snapshot;
  size_t args_bytes;   // expected sizeof(args)
};

extern std::atomic<unsigned long long> g_launches;
inline void count_launch(unsigned long long k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Per-app tables.  Each returns false when the id is not theirs.
bool mb_method_info(uint32_t id, MethodInfo* mi);
bool mb_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args);
bool mb_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok);

bool gol_method_info(uint32_t id, MethodInfo* mi);
bool gol_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args);
bool gol_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok);

bool wt_method_info(uint32_t id, MethodInfo* mi);
bool wt_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args);
bool wt_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok);
bool wt_ctor_launch(uint32_t id, const LaunchCtx& c, uint32_t T, uint64_t n, const void* args, size_t bytes, int* ok);

bool nb_method_info(uint32_t id, MethodInfo* mi);
bool nb_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args);
bool nb_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok);
bool nb_ctor_launch(uint32_t id, const LaunchCtx& c, uint32_t T, uint64_t n, const void* args, size_t bytes, int* ok);

// CTAs of `kernel` that are resident on one SM at `threads` threads (cached).
int resident_ctas(const void* kernel, int threads);

// Persistent grid: exactly one wave of resident CTAs (a multiple of the SM count).
template <typename K>
inline int persistent_grid(const LaunchCtx& c, K kernel, int threads = 256) {
  return resident_ctas((const void*)kernel, threads) * c.sms;
}
template <typename K>
inline int grid_for(const LaunchCtx& c, uint64_t n, K kernel, int threads = 256) {
  const uint64_t g = (n + threads - 1) / threads;
  const uint64_t p = (uint64_t)persistent_grid(c, kernel, threads);
  return (int)(g < 1 ? 1 : (g < p ? g : p));
}

// launch helper for element-loop method kernels
template <class Mth>
inline void launch_doall(const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  typename Mth::Args a = *reinterpret_cast<const typename Mth::Args*>(args);
  if (snapshot == 2) {                                                     // dynamic work distribution
    cudaMemsetAsync(&c.h.ctrl[CTRL_WORK], 0, 8, c.st);
    k_doall<Mth, kSchedDynamic><<<persistent_grid(c, k_doall<Mth, kSchedDynamic>), 256, 0, c.st>>>(c.h, T, 1, c.rk, a);
  } else if (snapshot == 3) {
    k_doall<Mth, kSchedBlocked><<<persistent_grid(c, k_doall<Mth, kSchedBlocked>), 256, 0, c.st>>>(c.h, T, 1, c.rk, a);
  } else {
    k_doall<Mth, kSchedCyclic><<<persistent_grid(c, k_doall<Mth, kSchedCyclic>), 256, 0, c.st>>>(c.h, T, snapshot, c.rk,
                                                                                                 a);
  }
  count_launch();
}

// quad-mapped body (k_doall_quad): snapshot 3 -> blocked distribution, else cyclic
template <class Mth>
inline void launch_doall_quad(const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  typename Mth::Args a = *reinterpret_cast<const typename Mth::Args*>(args);
  if (snapshot == 3)
    k_doall_quad<Mth, kSchedBlocked><<<persistent_grid(c, k_doall_quad<Mth, kSchedBlocked>), 256, 0, c.st>>>(c.h, T, 1, c.rk, a);
  else
    k_doall_quad<Mth, kSchedCyclic><<<persistent_grid(c, k_doall_quad<Mth, kSchedCyclic>), 256, 0, c.st>>>(c.h, T, snapshot ? 1 : 0,
                                                                                                           c.rk, a);
  count_launch();
}

// selective body (k_doall_sel): the iteration-bitmap snapshot, dynamic distribution
template <class Mth>
inline void launch_doall_sel(const LaunchCtx& c, uint32_t T, const void* args) {
  typename Mth::Args a = *reinterpret_cast<const typename Mth::Args*>(args);
  cudaMemsetAsync(&c.h.ctrl[CTRL_WORK], 0, 8, c.st);
  k_doall_sel<Mth><<<persistent_grid(c, k_doall_sel<Mth>), 256, 0, c.st>>>(c.h, T, c.rk, a);
  count_launch();
}

// block-mapped body (k_doall_block): one lane per block
template <class Mth>
inline void launch_doall_block(const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  typename Mth::Args a = *reinterpret_cast<const typename Mth::Args*>(args);
  k_doall_block<Mth><<<persistent_grid(c, k_doall_block<Mth>), 256, 0, c.st>>>(c.h, T, snapshot ? 1 : 0, c.rk, a);
  count_launch();
}

}  // namespace dsr
