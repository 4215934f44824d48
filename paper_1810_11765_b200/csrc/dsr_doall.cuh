// dsr_doall.cuh -- parallel do-all (§3.6, Alg. 5).
//
// Prologue (k_compact): one pass over the leaf containers of allocated[T]
// that (a) skips containers whose nested-level bit is 0, (b) counts
// set bits, prefix-sums them across the CTA (warp shuffles) and reserves a
// CTA-wide range of R with ONE atomicAdd (the paper's atomic cursor, P:641,
// at CTA rather than thread granularity), (c) writes R coalesced (lane j of a
// warp expands bit j / j+32 of a container) and (d) optionally snapshots the
// iteration bitmaps iter_bm[b] = alloc_bm[b] & valid(N_T) (C12).  The
// count r stays on the device (ctrl[CTRL_RCOUNT]); nothing returns to the host.
//
// Body (k_doall<Method>): a persistent grid strides over the r*N_T elements
// e -> block R[e / N_T], slot e % N_T (reading R-ASSIGN / C9: the paper's
// id_O / id_B formulas with an element stride, exact for every n).  Lanes of
// a warp take consecutive slots of a block, so every SOA field access of a
// warp is one contiguous column segment.
#pragma once
#include "dsr_device.cuh"

namespace dsr {

constexpr int kCompactThreads = 64;
#ifndef DSR_DOALL_CHUNK
#define DSR_DOALL_CHUNK 2
#endif
constexpr uint32_t kDoallChunk = DSR_DOALL_CHUNK;   // dynamic work unit of allocating passes: 2 x 32 elements per warp (sweep 1/2/4/8 -> 2)

static __global__ void __launch_bounds__(kCompactThreads) k_compact(DevHeap h, uint32_t T, int snapshot) {
  __shared__ uint64_t s_word[kCompactThreads];
  __shared__ uint32_t s_off[kCompactThreads];
  __shared__ uint32_t s_warp[kCompactThreads / 32];
  __shared__ uint32_t s_base;
  const DevBitmap& ab = h.allocbm[T];
  const uint64_t nwords = ((uint64_t)h.M + 63) / 64;
  const uint64_t i = (uint64_t)blockIdx.x * kCompactThreads + threadIdx.x;
  uint64_t w = 0;
  if (i < nwords) {
    bool any = true;
    if (ab.nlevels > 1) any = (ab.lvl[1][i >> 6] >> (i & 63)) & 1ull;    // hierarchical skip
    if (any) w = ab.lvl[0][i];
  }
  const uint32_t cnt = __popcll(w);
  // CTA exclusive scan of cnt
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += v;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int k = 0; k < kCompactThreads / 32; ++k) { const uint32_t t = s_warp[k]; s_warp[k] = run; run += t; }
    s_base = run ? atomicAdd((unsigned int*)&h.ctrl[CTRL_RCOUNT], run) : 0u;
  }
  __syncthreads();
  s_word[threadIdx.x] = w;
  s_off[threadIdx.x] = s_base + s_warp[wid] + inc - cnt;
  __syncwarp();
  // warp-cooperative expansion of this warp's 32 containers
  const uint64_t valid = h.types[T].valid;
  for (int k = 0; k < 32; ++k) {
    const uint32_t src = wid * 32 + k;
    const uint64_t wk = s_word[src];
    if (wk == 0) continue;
    const uint32_t off = s_off[src];
    const uint64_t cidx = (uint64_t)blockIdx.x * kCompactThreads + src;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const uint32_t bit = lane + 32 * half;
      if ((wk >> bit) & 1ull) {
        const uint32_t pos = off + __popcll(wk & ((1ull << bit) - 1ull));
        const uint32_t b = (uint32_t)(cidx * 64 + bit);
        h.R[pos] = b;
      }
    }
  }
  if (snapshot) {
    // iteration-bitmap snapshot of this warp's 2048 blocks as independent,
    // coalesced loads (a 256-B row of alloc_bm per warp and step, 8 rows in
    // flight): done inside the loop above, each container's load -> store
    // chain serialised the warp (Wa-Tor prologues 51 us with, 21 us without)
    const uint64_t b0 = ((uint64_t)blockIdx.x * kCompactThreads + wid * 32) * 64;
    for (int j0 = 0; j0 < 64; j0 += 8) {
      uint64_t v[8];
      bool on[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        on[u] = (s_word[wid * 32 + (j >> 1)] >> (lane + 32 * (j & 1))) & 1ull;
        v[u] = on[u] ? __ldg((const unsigned long long*)h.alloc_bm + b0 + 64 * (j >> 1) + lane + 32 * (j & 1)) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        if (on[u]) h.iter_bm[b0 + 64 * (j >> 1) + lane + 32 * (j & 1)] = v[u] & valid;
      }
    }
  }
}

// Persistent-grid element loop shared by all method kernels.  rk < 0: the
// whole of R; rk = k: the k-th type's range of a subtree do-all
// (ctrl[CTRL_RBEG + k] .. ctrl[CTRL_RBEG + k + 1]).
// SCHED: how elements are dealt to warps (all three visit every element once):
//   kSchedCyclic  grid stride -- all warps sweep R together (streaming passes)
//   kSchedDynamic warps take 32 x kDoallChunk elements from a device counter
//   kSchedBlocked each warp owns one contiguous range of R
enum { kSchedCyclic = 0, kSchedDynamic = 1, kSchedBlocked = 2 };
template <class Mth, int SCHED>
__global__ void __launch_bounds__(256, 8) k_doall(DevHeap h, uint32_t T, int snapshot, int rk, typename Mth::Args a) {
  uint32_t rb = 0, re;
  if (rk < 0) {
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RCOUNT]);
  } else {
    rb = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk]);
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk + 1]);
  }
  const uint32_t* R = h.R + rb;
  const uint32_t N = h.types[T].cap;
  const uint64_t total = (uint64_t)(re - rb) * N;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  typename Mth::Acc acc;
  if (SCHED == kSchedDynamic) {
    // Passes with very uneven per-object cost (several allocations per visit):
    // a warp takes the next 32 x kDoallChunk elements from a device counter
    // (ctrl[CTRL_WORK], zeroed before the launch) instead of a static stride --
    // no tail of idle SMs waiting for the slowest warps.  (Measured: GoL
    // Alive.update 19.5 -> 10-13 ms at 16384^2; light passes get slower.)
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t q32 = 32u / N, r32 = 32u % N;
    for (;;) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&h.ctrl[CTRL_WORK], 32ull * kDoallChunk);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= total) break;
      uint64_t e = base + lane;
      uint64_t bi = e / N;
      uint32_t s = (uint32_t)(e - bi * N);
      for (uint32_t k = 0; k < kDoallChunk && e < total; ++k, e += 32) {
        const uint32_t b = R[bi];
        if ((h.iter_bm[b] >> s) & 1ull) Mth::run(h, T, b, s, a, acc);
        bi += q32;
        s += r32;
        if (s >= N) { s -= N; ++bi; }
      }
    }
    Mth::flush(acc, a);
    return;
  }
  if (SCHED == kSchedBlocked) {
    // Passes that free whole blocks (every slot destroyed): with the cyclic
    // stride the whole grid works on one window of consecutive blocks, whose
    // FIRST / EMPTY transitions all hit the same few words of the active /
    // allocated / free bitmaps.  A contiguous range per warp puts concurrent
    // warps ~r/#warps blocks apart (measured: microbench drain 1.72 -> 1.32 ms;
    // lighter passes got slower, so it is opt-in per method).
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = stride >> 5, w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t C = (total + 31) >> 5, c0 = w * C / nw, c1 = (w + 1) * C / nw;
    const uint32_t q32 = 32u / N, r32 = 32u % N;
    uint64_t e = c0 * 32 + lane;
    uint64_t bi = e / N;
    uint32_t s = (uint32_t)(e - bi * N);
    for (uint64_t c = c0; c < c1; ++c, e += 32) {
      if (e < total) {
        const uint32_t b = R[bi];
        const uint64_t w = snapshot ? h.iter_bm[b] : ld_relaxed(h.alloc_bm + b);
        if ((w >> s) & 1ull) Mth::run(h, T, b, s, a, acc);
      }
      bi += q32;
      s += r32;
      if (s >= N) { s -= N; ++bi; }
    }
    Mth::flush(acc, a);
    return;
  }
  // element e -> (block index bi, slot s) = (e / N, e % N), advanced
  // incrementally by the grid stride (two divisions per thread, not per element)
  uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t bi = e / N;
  uint32_t s = (uint32_t)(e - bi * N);
  const uint64_t dbi = stride / N;
  const uint32_t ds = (uint32_t)(stride - dbi * N);
  for (; e < total; e += stride) {
    const uint32_t b = R[bi];
    const uint64_t w = snapshot ? h.iter_bm[b] : ld_relaxed(h.alloc_bm + b);
    if ((w >> s) & 1ull) Mth::run(h, T, b, s, a, acc);
    bi += dbi;
    s += ds;
    if (s >= N) { s -= N; ++bi; }
  }
  Mth::flush(acc, a);
}

// Quad-mapped do-all body (vectorised, reading C31): element e is
// the quad of slots 4q .. 4q+3 of block R[e / Q], Q = ceil(N_T / 4), so a warp
// covers 128 consecutive slots and a u32 column segment of a quad is one
// 16-B aligned 128-bit load (columns are 16-B aligned, R-LAYOUT).  The method
// gets the quad's live-slot mask m4 (bit j = slot 4q + j visited; padding and
// slots beyond N_T are never set) and must store only to visited slots (C31).
// Grid-stride over the quads with an incremental (block, quad) pair.
template <class Mth, int SCHED>
__global__ void __launch_bounds__(256) k_doall_quad(DevHeap h, uint32_t T, int snapshot, int rk, typename Mth::Args a) {
  uint32_t rb = 0, re;
  if (rk < 0) {
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RCOUNT]);
  } else {
    rb = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk]);
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk + 1]);
  }
  const uint32_t* R = h.R + rb;
  const uint32_t Q = (h.types[T].cap + 3) >> 2;
  const uint64_t valid = h.types[T].valid;
  const uint64_t total = (uint64_t)(re - rb) * Q;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  typename Mth::Acc acc;
  // kSchedCyclic: grid stride; kSchedBlocked: each warp owns one contiguous
  // range of quads (passes that free whole blocks: concurrent warps then work
  // on blocks far apart, so their block transitions hit different bitmap words)
  uint64_t e, step, end;
  if (SCHED == kSchedBlocked) {
    const uint64_t nw = stride >> 5, w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t C = (total + 31) >> 5;
    e = (w * C / nw) * 32 + (threadIdx.x & 31);
    end = ((w + 1) * C / nw) * 32;
    step = 32;
  } else {
    e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    end = total;
    step = stride;
  }
  if (end > total) end = total;
  uint64_t bi = e / Q;
  uint32_t q = (uint32_t)(e - bi * Q);
  const uint64_t dbi = step / Q;
  const uint32_t dq = (uint32_t)(step - dbi * Q);
  for (; e < end; e += step) {
    const uint32_t b = __ldg(R + bi);
    const uint64_t w = snapshot ? __ldg((const unsigned long long*)h.iter_bm + b) : (ld_relaxed(h.alloc_bm + b) & valid);
    const uint32_t m4 = (uint32_t)(w >> (4 * q)) & 0xFu;
    if (m4) Mth::run4(h, T, b, q, m4, a, acc);
    bi += dbi;
    q += dq;
    if (q >= Q) { q -= Q; ++bi; }
  }
  Mth::flush(acc, a);
}

// the quad q of a u32 column f: one aligned 16-B segment (4 slots)
__device__ __forceinline__ uint4* quad_u32(const DevHeap& h, uint32_t T, uint32_t f, uint32_t b, uint32_t q) {
  return reinterpret_cast<uint4*>(h.data + (size_t)b * h.block_bytes + h.types[T].col_off[f] + 16u * q);
}

// Method helpers: most methods keep no per-thread accumulator.
struct NoAcc {};
#define DSR_NO_ACC                                                        \
  typedef NoAcc Acc;                                                      \
  static __device__ __forceinline__ void flush(Acc&, const Args&) {}

// Per-thread event counters flushed with one warp-aggregated atomic per lane
// group (used by Wa-Tor / N-body for born/eaten/starved/merged counts).
struct Counters4 {
  uint32_t c[4];
  __device__ Counters4() : c{0, 0, 0, 0} {}
};
__device__ __forceinline__ void flush_counters4(Counters4& acc, unsigned long long* out) {
  if (!out) return;
  const uint32_t act = __activemask();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t v = __reduce_add_sync(act, acc.c[k]);
    if (v && lane_id() == (uint32_t)(__ffs(act) - 1)) atomicAdd(out + k, (unsigned long long)v);
  }
}

}  // namespace dsr
