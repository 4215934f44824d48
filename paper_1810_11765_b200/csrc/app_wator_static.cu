// app_wator_static.cu -- the paper's static-allocation baseline of Wa-Tor
// ("Baselines (SOA/AOS) are application variants without any
// dynamic memory allocation ... In category (3), classes are merged with the
// underlying static cell data structure, which wastes memory in case of empty
// cells").  Same rules, same keys and the same request / decide protocol as
// the object version (app_wator.cu, reading R-WATOR), on cell-indexed SOA
// arrays: kind u8, egg u32, energy u32, target u32, req u8.  It exists to
// price DynaSOAr's dynamic allocation on B200; results
// are identical to the object version and the oracle.
//
// Per half step (fish, then sharks) three kernels:
//   prepare  every agent of the moving kind: egg += 1, target := own cell
//            (marks it as a snapshot agent), sharks lose one energy; then a
//            request bit into the chosen neighbour cell (byte atomicOr) or a
//            "stay" bit on its own cell.
//   decide   every cell with requests and no stay bit grants one requester
//            (target[requester] := cell); then clears its request byte, so
//            the next prepare starts from zero without a memset.
//   update   every snapshot agent (target != NONE) starves, stays or moves,
//            eats a fish on arrival (sharks) and leaves a newborn behind.
// Only the arrival cell's owner grants a move, so every write has one writer.
#include "dsr_host.h"

namespace dsr {

constexpr uint32_t kWsNone = 0xFFFFFFFFu;
enum { WS_EMPTY = 0, WS_FISH = 1, WS_SHARK = 2 };

__device__ __forceinline__ uint32_t ws_nbr(uint32_t W, uint32_t H, uint32_t c, uint32_t d) {
  const uint32_t x = c % W, y = c / W;
  switch (d) {
    case 0: return (y == 0 ? H - 1 : y - 1) * W + x;
    case 1: return y * W + (x + 1 == W ? 0 : x + 1);
    case 2: return (y + 1 == H ? 0 : y + 1) * W + x;
    default: return y * W + (x == 0 ? W - 1 : x - 1);
  }
}
// byte atomicOr through the aligned 32-bit word (the req array is padded to 4 B)
__device__ __forceinline__ void ws_req_set(uint8_t* req, uint32_t c, uint32_t bit) {
  atomicOr(reinterpret_cast<unsigned int*>(req + (c & ~3u)), (1u << bit) << (8 * (c & 3u)));
}

template <int ME>
__global__ void __launch_bounds__(256) k_ws_prepare(dsr_wator_static_args a, uint32_t step) {
  const uint32_t N = a.W * a.H;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    if (a.kind[c] != ME) continue;
    a.egg[c] += 1;
    a.target[c] = c;
    if (ME == WS_SHARK) {
      const uint32_t en = a.energy[c] - 1;
      a.energy[c] = en;
      if (en == 0) continue;                                     // starves in update
    }
    uint32_t fd[4], nfd = 0, fr[4], nfr = 0;
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d) {
      const uint8_t k = a.kind[ws_nbr(a.W, a.H, c, d)];
      if (k == WS_FISH) fd[nfd++] = d;
      if (k == WS_EMPTY) fr[nfr++] = d;
    }
    const uint64_t key = rng_key(a.seed, step, ME == WS_FISH ? 1 : 3, c);
    int d = -1;
    if (ME == WS_SHARK && nfd) d = (int)fd[(uint32_t)((key >> 32) % nfd)];
    else if (nfr) d = (int)fr[(uint32_t)((key >> 32) % nfr)];
    if (d >= 0) ws_req_set(a.req, ws_nbr(a.W, a.H, c, (uint32_t)d), (uint32_t)d ^ 2u);
    else ws_req_set(a.req, c, 4);
  }
}

template <int ME>
__global__ void __launch_bounds__(256) k_ws_decide(dsr_wator_static_args a, uint32_t step) {
  const uint32_t N = a.W * a.H;
  // four cells per thread: one 32-bit load of their request bytes
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; 4 * q < N; q += gridDim.x * blockDim.x) {
    const uint32_t r4 = reinterpret_cast<const uint32_t*>(a.req)[q];
    if (r4 == 0) continue;
    reinterpret_cast<uint32_t*>(a.req)[q] = 0;
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
      const uint32_t r = (r4 >> (8 * j)) & 0x1Fu, c = 4 * q + j;
      if (r == 0 || (r & 0x10u) || c >= N) continue;
      uint32_t D[4], nd = 0;
#pragma unroll
      for (uint32_t d = 0; d < 4; ++d)
        if (r & (1u << d)) D[nd++] = d;
      const uint32_t d = D[(uint32_t)((rng_key(a.seed, step, ME == WS_FISH ? 2 : 4, c) >> 32) % nd)];
      a.target[ws_nbr(a.W, a.H, c, d)] = c;
    }
  }
}

template <int ME>
__global__ void __launch_bounds__(256) k_ws_update(dsr_wator_static_args a) {
  const uint32_t N = a.W * a.H;
  uint32_t born = 0, eaten = 0, starved = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    const uint32_t t = a.target[c];
    if (t == kWsNone) continue;                                   // not an agent of this half step
    a.target[c] = kWsNone;
    if (ME == WS_SHARK && a.energy[c] == 0) {
      a.kind[c] = WS_EMPTY; a.egg[c] = 0;
      ++starved;
      continue;
    }
    if (t == c) continue;
    const uint32_t egg = a.egg[c];
    uint32_t en = ME == WS_SHARK ? a.energy[c] : 0u;
    if (ME == WS_SHARK && a.kind[t] == WS_FISH) { ++eaten; en = a.SS; }
    a.kind[t] = ME; a.egg[t] = egg; a.energy[t] = en;
    if (egg >= (ME == WS_FISH ? a.FB : a.SB)) {                   // newborn on the old cell
      a.egg[t] = 0;
      a.egg[c] = 0; a.energy[c] = ME == WS_SHARK ? a.SS : 0u;
      ++born;
    } else {
      a.kind[c] = WS_EMPTY; a.egg[c] = 0; a.energy[c] = 0;
    }
  }
  if (a.counters) {
    const uint32_t act = __activemask();
    const uint32_t b = __reduce_add_sync(act, born), e = __reduce_add_sync(act, eaten), s = __reduce_add_sync(act, starved);
    if (lane_id() == (uint32_t)(__ffs(act) - 1)) {
      if (b) atomicAdd(&a.counters[ME == WS_FISH ? 0 : 1], (unsigned long long)b);
      if (e) atomicAdd(&a.counters[2], (unsigned long long)e);
      if (s) atomicAdd(&a.counters[3], (unsigned long long)s);
    }
  }
}

static int ws_grid(const void* k, int sms) { return resident_ctas(k, 256) * sms; }

}  // namespace dsr

using namespace dsr;

extern "C" dsr_status dsr_wator_static_step(const dsr_wator_static_args* args, uint32_t steps, void* stream) {
  if (!args) return DSR_ERR_INVALID;
  const dsr_wator_static_args a = *args;
  if (a.W < 3 || a.H < 3 || (uint64_t)a.W * a.H >= 0xFFFFFFFFull || !a.kind || !a.egg || !a.energy || !a.target ||
      !a.req || a.FB == 0 || a.SB == 0 || a.SS == 0)
    return DSR_ERR_INVALID;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return DSR_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  for (uint32_t i = 0; i < steps; ++i) {
    const uint32_t step = a.step + i;
    k_ws_prepare<WS_FISH><<<ws_grid((const void*)k_ws_prepare<WS_FISH>, sms), 256, 0, st>>>(a, step);
    k_ws_decide<WS_FISH><<<ws_grid((const void*)k_ws_decide<WS_FISH>, sms), 256, 0, st>>>(a, step);
    k_ws_update<WS_FISH><<<ws_grid((const void*)k_ws_update<WS_FISH>, sms), 256, 0, st>>>(a);
    k_ws_prepare<WS_SHARK><<<ws_grid((const void*)k_ws_prepare<WS_SHARK>, sms), 256, 0, st>>>(a, step);
    k_ws_decide<WS_SHARK><<<ws_grid((const void*)k_ws_decide<WS_SHARK>, sms), 256, 0, st>>>(a, step);
    k_ws_update<WS_SHARK><<<ws_grid((const void*)k_ws_update<WS_SHARK>, sms), 256, 0, st>>>(a);
    count_launch(6);
  }
  return cudaPeekAtLastError() == cudaSuccess ? DSR_OK : DSR_ERR_CUDA;
}
