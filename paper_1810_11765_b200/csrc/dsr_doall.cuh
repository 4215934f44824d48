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

#ifndef DSR_DOALL_CHUNK
#define DSR_DOALL_CHUNK 2
#endif
constexpr uint32_t kDoallChunk = DSR_DOALL_CHUNK;   // dynamic work unit of allocating passes: 2 x 32 elements per warp (sweep 1/2/4/8 -> 2)
constexpr int kCompactThreads = 256;

// Prologue driven from the nested level (Alg. 5's recursion, and
// the paper's atomic cursor), so its cost follows the allocated blocks,
// not the heap size M: a persistent grid of warps strides over the
// halves of the level-1 containers of allocated[T]; a zero half (32 leaf
// words, 2048 blocks) costs one load.  For a non-zero one, lane l reads leaf
// word l (only if its level-1 bit is set), the warp prefix-sums the
// popcounts, reserves its range of R with ONE atomicAdd, and expands the leaf
// words into R cooperatively (lane j writes bit j / j + 32 of each word:
// coalesced).  snapshot: iter_bm[b] = alloc_bm[b] & valid(N_T) for the same
// blocks (C12) as a separate batch of independent coalesced loads (inside
// the expansion each word's load -> store chain would serialise the warp).
// The count r stays on the device (ctrl[CTRL_RCOUNT]).
static __global__ void __launch_bounds__(kCompactThreads) k_compact(DevHeap h, uint32_t T, int snapshot) {
  const DevBitmap& ab = h.allocbm[T];
  const uint64_t nwords = ((uint64_t)h.M + 63) / 64;
  const uint64_t n1 = (nwords + 63) / 64;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t valid = h.types[T].valid;
  // work item = half a level-1 container: 32 leaf words, lane l <-> leaf word l
  for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < 2 * n1; it += nw) {
    const uint64_t i1 = it >> 1;
    const uint32_t half = (uint32_t)(it & 1);
    uint64_t w1;
    if (ab.nlevels > 1) {
      w1 = __ldg((const unsigned long long*)ab.lvl[1] + i1);
    } else {                                                       // one level: every leaf word (nwords <= 64)
      w1 = nwords >= 64 ? ~0ull : ((1ull << nwords) - 1ull);
    }
    const uint32_t w32 = (uint32_t)(w1 >> (32 * half));
    if (w32 == 0) continue;
    const uint64_t word = i1 * 64 + 32 * half + lane;
    const uint64_t wl = ((w32 >> lane) & 1u) ? __ldg((const unsigned long long*)ab.lvl[0] + word) : 0ull;
    const uint32_t c = __popcll(wl);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd((unsigned int*)&h.ctrl[CTRL_RCOUNT], total);
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t off = base + incl - c;
    const uint32_t srcs = __ballot_sync(0xffffffffu, wl != 0);
    // expansion: leaf word k -> its blocks, lane j takes bits j and j + 32 (coalesced R stores)
    uint32_t m = srcs;
    while (m) {
      const uint32_t k = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t wk = shfl64(0xffffffffu, wl, k);
      const uint32_t ok = __shfl_sync(0xffffffffu, off, k);
      const uint64_t bw = (i1 * 64 + 32 * half + k) * 64;                // first block of leaf word k
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t bit = lane + 32 * hh;
        if ((wk >> bit) & 1ull) h.R[ok + __popcll(wk & ((1ull << bit) - 1ull))] = (uint32_t)(bw + bit);
      }
    }
    if (snapshot) {
      // iteration bitmaps of the same blocks: rows of 32 consecutive u64,
      // 8 leaf words' loads in flight before their stores
      m = srcs;
      while (m) {
        uint64_t v[8][2], wkk[8];
        uint32_t ks[8];
        uint32_t n = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          ks[u] = m ? (uint32_t)(__ffs(m) - 1) : 0u;
          if (m) { m &= m - 1; n = u + 1; }
          wkk[u] = shfl64(0xffffffffu, wl, ks[u]);
          if ((uint32_t)u >= n) wkk[u] = 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint64_t bw = (i1 * 64 + 32 * half + ks[u]) * 64;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t bit = lane + 32 * hh;
            v[u][hh] = ((wkk[u] >> bit) & 1ull) ? __ldg((const unsigned long long*)h.alloc_bm + bw + bit) : 0ull;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint64_t bw = (i1 * 64 + 32 * half + ks[u]) * 64;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t bit = lane + 32 * hh;
            if ((wkk[u] >> bit) & 1ull) h.iter_bm[bw + bit] = v[u][hh] & valid;
          }
        }
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
#ifndef DSR_DOALL_MINB
#define DSR_DOALL_MINB 8
#endif
template <class Mth, int SCHED>
__global__ void __launch_bounds__(256, DSR_DOALL_MINB) k_doall(DevHeap h, uint32_t T, int snapshot, int rk, typename Mth::Args a) {
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

// Selective do-all body, for methods that do real work on a minority of
// their objects (Mth::select(h, T, b, s, a): a cheap test, e.g. "my action is
// not NONE"; Mth::run only where it holds).  A warp takes 32 x kDoallChunk
// elements at a time from a device counter (dynamic distribution), tests them
// with full warps, appends the selected (block, slot) pairs to its queue in
// shared memory (ballot + popc), and whenever 32 are queued runs the method
// on them with all 32 lanes: the allocations and destroys of the body then
// coalesce over 32 objects instead of the few a warp's slots happen to select
// (GoL's update passes ran at 6-8 active threads per instruction).
template <class Mth>
__global__ void __launch_bounds__(256) k_doall_sel(DevHeap h, uint32_t T, int rk, typename Mth::Args a) {
  __shared__ unsigned long long s_q[8][64];
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
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  unsigned long long* const q = s_q[threadIdx.x >> 5];
  uint32_t cnt = 0;
  typename Mth::Acc acc;
  const uint32_t q32 = 32u / N, r32 = 32u % N;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&h.ctrl[CTRL_WORK], 32ull * kDoallChunk);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= total) break;
    uint64_t e = base + lane;
    uint64_t bi = e / N;
    uint32_t s = (uint32_t)(e - bi * N);
    for (uint32_t k = 0; k < kDoallChunk; ++k, e += 32) {
      bool sel = false;
      uint32_t b = 0;
      if (e < total) {
        b = R[bi];
        sel = ((h.iter_bm[b] >> s) & 1ull) && Mth::select(h, T, b, s, a);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      if (sel) q[cnt + __popc(bal & lt)] = ((unsigned long long)b << 6) | s;
      cnt += __popc(bal);
      __syncwarp();
      if (cnt >= 32) {                                     // a full warp of work
        cnt -= 32;
        const unsigned long long it = q[cnt + lane];
        __syncwarp();
        Mth::run(h, T, (uint32_t)(it >> 6), (uint32_t)(it & 63), a, acc);
      }
      bi += q32;
      s += r32;
      if (s >= N) { s -= N; ++bi; }
    }
  }
  if (lane < cnt) {
    const unsigned long long it = q[lane];
    Mth::run(h, T, (uint32_t)(it >> 6), (uint32_t)(it & 63), a, acc);
  }
  Mth::flush(acc, a);
}

// Block-mapped do-all body: one lane per block of R, for methods whose work
// on a block's visited objects combines into one action per block (destroying
// all of them is one atomicAnd of the block's bitmap: the coalescing of
// P:649 taken to the whole block).  The method gets the block's visited-slot
// mask w (snapshot: iteration bitmap, else allocation bitmap & valid).  Each
// warp owns one contiguous range of R (blocked) and each lane one contiguous
// sub-range of it, so the 32 lanes' block transitions hit bitmap words far
// apart and every lane keeps its own chain of dependent atomics in flight.
template <class Mth>
__global__ void __launch_bounds__(256) k_doall_block(DevHeap h, uint32_t T, int snapshot, int rk, typename Mth::Args a) {
  uint32_t rb = 0, re;
  if (rk < 0) {
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RCOUNT]);
  } else {
    rb = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk]);
    re = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RBEG + rk + 1]);
  }
  const uint32_t* R = h.R + rb;
  const uint64_t valid = h.types[T].valid;
  const uint64_t nb = re - rb;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5, w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w0 = w * nb / nw, w1 = (w + 1) * nb / nw;
  const uint64_t i0 = w0 + (w1 - w0) * lane / 32, i1 = w0 + (w1 - w0) * (lane + 1) / 32;
  typename Mth::Acc acc;
  for (uint64_t i = i0; i < i1; ++i) {
    const uint32_t b = __ldg(R + i);
    const uint64_t m = snapshot ? __ldg((const unsigned long long*)h.iter_bm + b) : (ld_relaxed(h.alloc_bm + b) & valid);
    if (m) Mth::runb(h, T, b, m, a, acc);
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
