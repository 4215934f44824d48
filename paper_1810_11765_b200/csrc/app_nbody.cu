// app_nbody.cu -- N-body with collisions (Table 1, Listing 1 P:143-183;
// reading R-NBODY).  Type 0 = Body{x, y, vx, vy, fx, fy, m: f32; id, target,
// incoming: u32; merged: u8} (41 B, N_T = 64).
//
// device_do -- the sequential all-bodies loop inside each
// body's method -- becomes a tiled all-pairs gather over an id-indexed SOA
// snapshot S (x, y, m) written by the preceding snapshot do-all: each CTA
// stages 256 snapshot entries in shared memory and every thread sums its
// body's interactions tile by tile in id order (the paper's terms, a fixed
// deterministic order).  Dead ids have m = 0 in S and contribute 0.
// Merge bookkeeping (target / incoming) lives in id-indexed arrays so that the
// same kernels serve one GPU and an id-range-sharded multi-GPU run (where S,
// V and target are all-gathered between passes).
#include <algorithm>
#include <cstring>
#include <cuda.h>   // cuStreamWaitValue32 (types only: resolved at run time)
#include "dsr_host.h"

namespace dsr {

enum { NB_X = 0, NB_Y, NB_VX, NB_VY, NB_FX, NB_FY, NB_M, NB_ID, NB_TARGET, NB_INCOMING, NB_MERGED };
constexpr uint32_t kNone = 0xFFFFFFFFu;

template <class V>
__device__ __forceinline__ V& bf(const DevHeap& h, uint32_t b, uint32_t s, int f) {
  return *field_ptr<V>(h, 0, (uint32_t)f, b, s);
}
__device__ __forceinline__ float4 s4(const dsr_nbody_args& a, uint32_t id) {
  return __ldg(reinterpret_cast<const float4*>(a.S) + id);
}

// ---- parallel_new<Body>(n): body i gets id id_lo + i
__global__ void __launch_bounds__(256) k_nb_new(DevHeap h, uint64_t n, dsr_nbody_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    const uint64_t nh = dsr_new_bulk(h, 0, i < n);
    if (!nh) continue;
    const uint32_t b = h_bid(nh), s = h_slot(nh);
    bf<float>(h, b, s, NB_X) = a.x0[i];
    bf<float>(h, b, s, NB_Y) = a.y0[i];
    bf<float>(h, b, s, NB_VX) = a.vx0[i];
    bf<float>(h, b, s, NB_VY) = a.vy0[i];
    bf<float>(h, b, s, NB_FX) = 0.f;
    bf<float>(h, b, s, NB_FY) = 0.f;
    bf<float>(h, b, s, NB_M) = a.m0[i];
    bf<uint32_t>(h, b, s, NB_ID) = a.id_lo + (uint32_t)i;
    bf<uint32_t>(h, b, s, NB_TARGET) = kNone;
    bf<uint32_t>(h, b, s, NB_INCOMING) = kNone;
    bf<uint8_t>(h, b, s, NB_MERGED) = 0;
  }
}

__global__ void k_nb_clear(uint64_t n, dsr_nbody_args a) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    a.shandle[i] = 0;
    a.incoming[i] = kNone;
    if (!a.npeers) {
      reinterpret_cast<float4*>(a.S)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.target[i] = kNone;
    } else if (i >= a.id_lo && i < a.id_hi) {
      // peer mode: only my rows -- the others' rows of S and target are theirs
      // to write (their pushes may already have arrived); mine are cleared in
      // every peer's S as well
      reinterpret_cast<float4*>(a.S)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.target[i] = kNone;
      for (uint32_t p = 0; p < a.npeers; ++p) reinterpret_cast<float4*>(a.peer_S[p])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}
// peer mode: this rank's rows of the epoch are in every peer (kernel boundary:
// the previous kernels' stores are performed) -> their flag slot `slot0 + rank`
__global__ void k_nb_signal(dsr_nbody_args a, uint32_t slot0) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence_system();
    for (uint32_t p = 0; p < a.npeers; ++p)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.peer_flags[p] + slot0 + a.rank), "r"(a.epoch + 1u)
                   : "memory");
  }
}
// peer mode: this rank's rows of target into every peer's target
__global__ void k_nb_push_target(dsr_nbody_args a) {
  for (uint32_t i = a.id_lo + blockIdx.x * blockDim.x + threadIdx.x; i < a.id_hi; i += gridDim.x * blockDim.x) {
    const uint32_t t = a.target[i];
    for (uint32_t p = 0; p < a.npeers; ++p) a.peer_target[p][i] = t;
  }
}

struct NbSnapshot {
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t id = bf<uint32_t>(h, b, s, NB_ID);
    const float4 p = make_float4(bf<float>(h, b, s, NB_X), bf<float>(h, b, s, NB_Y), bf<float>(h, b, s, NB_M), 0.f);
    const float2 v = make_float2(bf<float>(h, b, s, NB_VX), bf<float>(h, b, s, NB_VY));
    reinterpret_cast<float4*>(a.S)[id] = p;
    reinterpret_cast<float2*>(a.V)[id] = v;
    a.shandle[id] = make_handle(0, h.types[0].cap, b, s);
    // peer mode: the all-gather is this pass's stores into every peer's
    // snapshot (over NVLink when they are other GPUs) -- one kernel computes
    // the snapshot and distributes it
    for (uint32_t q = 0; q < a.npeers; ++q) {
      reinterpret_cast<float4*>(a.peer_S[q])[id] = p;
      reinterpret_cast<float2*>(a.peer_V[q])[id] = v;
    }
  }
};

// ---- device_do all-pairs gathers (force, merge search) -------------------
// Grid (i-blocks of 256 own ids, j-chunks of kChunk ids); a 128-thread CTA
// handles 2 bodies per thread and stages 256 snapshot entries per tile in
// shared memory.  Each (i, chunk) partial is written to scratch and a second
// kernel combines the chunks in increasing order: a fixed summation order that
// does not depend on the launch shape or on the number of GPUs.
constexpr uint32_t kChunk = 4096;
constexpr int kPairThreads = 128;

// Blackwell packed FP32 (f32x2: FADD2 / FMUL2 / FFMA2 on sm_100a): the two
// bodies of a thread go through one instruction per step; element-wise the
// operations and their order are exactly the scalar ones below, so results
// are bit-identical to a scalar evaluation.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void upk2(f32x2 r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r; asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r; asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r; asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}

// kNbPairs packed body pairs per thread (2 x kNbPairs bodies): every tile
// entry loaded from shared memory serves 2 x kNbPairs bodies, and the pairs'
// dependency chains interleave (per body the operations and their order are
// unchanged, so results do not depend on kNbPairs)
#ifndef DSR_NB_PAIRS
#define DSR_NB_PAIRS 2
#endif
constexpr int kNbPairs = DSR_NB_PAIRS;
constexpr uint32_t kIBlock = 256u * kNbPairs;       // bodies per CTA (i-block)
constexpr uint32_t kIBlocksPerChunk = kChunk / kIBlock;

// ---- the live list: both sides of the all-pairs passes run over the bodies
// that exist (device_do visits the Body objects), not over the whole id
// space -- the merges take 65,536 bodies down to ~18 k over the 1000 steps.
// Each 4096-id chunk c of S is compacted to its ids with m > 0, in ascending
// id order, as (x, y, m, id bits) at live[4 (4096 c + k)], count at cnt[c].
// A chunk's partial sum over its live bodies adds the same non-zero terms in
// the same order as the sum over all its ids (an empty id has m = 0 and adds
// exactly 0), so results do not change.
__device__ __forceinline__ float4* live_s(const dsr_nbody_args& a) { return reinterpret_cast<float4*>(a.live); }
__device__ __forceinline__ uint32_t* live_n(const dsr_nbody_args& a) {
  return reinterpret_cast<uint32_t*>(a.live + 4ull * a.n_total);
}
constexpr int kLiveThreads = kChunk / 4;
__global__ void __launch_bounds__(kLiveThreads) k_nb_live(dsr_nbody_args a) {
  __shared__ uint32_t s_w[kLiveThreads / 32];
  const uint32_t base = blockIdx.x * kChunk, end = min(base + kChunk, a.n_total);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float4 v[4];
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {                     // ids base + 4 t .. base + 4 t + 3, in order
    const uint32_t id = base + 4u * threadIdx.x + k;
    v[k] = id < end ? s4(a, id) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (v[k].z > 0.f) bits |= 1u << k;
  }
  const uint32_t cnt = __popc(bits);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) s_w[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += t;
    }
    s_w[lane] = x;                                   // inclusive warp totals
  }
  __syncthreads();
  uint32_t off = (wid ? s_w[wid - 1] : 0u) + incl - cnt;
  float4* out = live_s(a) + base;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((bits >> k) & 1u) out[off++] = make_float4(v[k].x, v[k].y, v[k].z, __uint_as_float(base + 4u * threadIdx.x + k));
  if (threadIdx.x == 0) live_n(a)[blockIdx.x] = s_w[kLiveThreads / 32 - 1];
}
// the i side of a CTA: live-list chunk ic = id_lo / 4096 + blockIdx.x / kIBlocksPerChunk,
// positions (blockIdx.x % kIBlocksPerChunk) * kIBlock + threadIdx.x + 128 m
struct PairI {
  uint32_t ic, pos0, n;
  __device__ PairI(const dsr_nbody_args& a)
      : ic(a.id_lo / kChunk + blockIdx.x / kIBlocksPerChunk),
        pos0((blockIdx.x % kIBlocksPerChunk) * kIBlock + threadIdx.x),
        n(live_n(a)[a.id_lo / kChunk + blockIdx.x / kIBlocksPerChunk]) {}
  // body m (0 .. 2 kNbPairs - 1) of this thread; id = 0xFFFFFFFF if none (or not mine)
  __device__ __forceinline__ float4 body(const dsr_nbody_args& a, int m, uint32_t& id) const {
    const uint32_t pos = pos0 + 128u * m;
    id = 0xFFFFFFFFu;
    if (pos >= n) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 p = __ldg(live_s(a) + (size_t)ic * kChunk + pos);
    const uint32_t i = __float_as_uint(p.w);
    if (i < a.id_lo || i >= a.id_hi) return make_float4(0.f, 0.f, 0.f, 0.f);
    id = i;
    return p;
  }
  __device__ __forceinline__ bool empty() const { return pos0 - threadIdx.x >= n; }   // CTA-uniform
};

__global__ void __launch_bounds__(kPairThreads) k_nb_force_part(dsr_nbody_args a) {
  __shared__ float4 tile[256];
  const uint32_t nl = a.id_hi - a.id_lo;
  const PairI I(a);
  if (I.empty()) return;                             // no body of this i-block exists
  const float eps2 = a.eps * a.eps;
  const f32x2 E2 = pk2(eps2, eps2);
  f32x2 PX[kNbPairs], PY[kNbPairs], AX[kNbPairs], AY[kNbPairs];
  uint32_t ID[2 * kNbPairs];
#pragma unroll
  for (int q = 0; q < kNbPairs; ++q) {
    const float4 p0 = I.body(a, 2 * q, ID[2 * q]), p1 = I.body(a, 2 * q + 1, ID[2 * q + 1]);
    PX[q] = pk2(p0.x, p1.x);
    PY[q] = pk2(p0.y, p1.y);
    AX[q] = pk2(0.f, 0.f);
    AY[q] = pk2(0.f, 0.f);
  }
  const uint32_t jc = blockIdx.y, nj = live_n(a)[jc];
  const float4* J = live_s(a) + (size_t)jc * kChunk;
  for (uint32_t j0 = 0; j0 < nj; j0 += 256) {
    __syncthreads();
    const uint32_t ja = j0 + threadIdx.x, jb = ja + 128;
    tile[threadIdx.x] = ja < nj ? __ldg(J + ja) : make_float4(0.f, 0.f, 0.f, 0.f);   // padding: m = 0
    tile[threadIdx.x + 128] = jb < nj ? __ldg(J + jb) : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 256; ++k) {
      const float4 p = tile[k];                      // padding entries have m = 0: they add exactly 0
      const f32x2 JX = pk2(p.x, p.x), JY = pk2(p.y, p.y), JM = pk2(p.z, p.z);
#pragma unroll
      for (int q = 0; q < kNbPairs; ++q) {
        // per body: dx = x_j - x_i, r = dx^2 + (dy^2 + eps^2), w = ((m_j v) v) v with
        // v = rsqrt(r), a += dx w  (P:171-174 with Plummer softening, R-NBODY)
        const f32x2 DX = sub2(JX, PX[q]), DY = sub2(JY, PY[q]);
        const f32x2 R = fma2(DX, DX, fma2(DY, DY, E2));
        float r0, r1;
        upk2(R, r0, r1);
        const f32x2 V = pk2(rsqrtf(r0), rsqrtf(r1));
        const f32x2 W = mul2(mul2(mul2(JM, V), V), V);
        AX[q] = fma2(DX, W, AX[q]);
        AY[q] = fma2(DY, W, AY[q]);
      }
    }
  }
  float2* part = reinterpret_cast<float2*>(a.scratch) + (size_t)blockIdx.y * nl;
#pragma unroll
  for (int q = 0; q < kNbPairs; ++q) {
    float ax0, ax1, ay0, ay1;
    upk2(AX[q], ax0, ax1);
    upk2(AY[q], ay0, ay1);
    if (ID[2 * q] != 0xFFFFFFFFu) part[ID[2 * q] - a.id_lo] = make_float2(ax0, ay0);
    if (ID[2 * q + 1] != 0xFFFFFFFFu) part[ID[2 * q + 1] - a.id_lo] = make_float2(ax1, ay1);
  }
}

// f_i = G m_i sum_j m_j (p_j - p_i) / (|p_j - p_i|^2 + eps^2)^{3/2}, chunks summed in order
__global__ void k_nb_force_sum(DevHeap h, dsr_nbody_args a) {
  const uint32_t nl = a.id_hi - a.id_lo, chunks = (a.n_total + kChunk - 1) / kChunk;
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < nl; li += gridDim.x * blockDim.x) {
    const uint64_t hd = a.shandle[a.id_lo + li];
    if (!hd) continue;
    float ax = 0.f, ay = 0.f;
    for (uint32_t c = 0; c < chunks; ++c) {
      const float2 v = reinterpret_cast<const float2*>(a.scratch)[(size_t)c * nl + li];
      ax += v.x;
      ay += v.y;
    }
    const uint32_t b = h_bid(hd), s = h_slot(hd);
    const float gm = __fmul_rn(a.G, bf<float>(h, b, s, NB_M));
    bf<float>(h, b, s, NB_FX) = __fmul_rn(gm, ax);
    bf<float>(h, b, s, NB_FY) = __fmul_rn(gm, ay);
  }
}

// Per-body arithmetic with explicit rounding (no FMA contraction), so the
// heap version and the static baseline below perform identical operations
// whatever the compiler contracts in each kernel (bit-exact comparison).
__device__ __forceinline__ float nb_step_v(float v, float f, float m, float dt) {
  return __fadd_rn(v, __fmul_rn(__fdiv_rn(f, m), dt));
}
__device__ __forceinline__ float nb_step_p(float p, float v, float dt) { return __fadd_rn(p, __fmul_rn(v, dt)); }
__device__ __forceinline__ float nb_mix(float m, float u, float mi, float ui, float mn) {
  return __fdiv_rn(__fadd_rn(__fmul_rn(m, u), __fmul_rn(mi, ui)), mn);
}

struct NbMove {   // semi-implicit Euler, velocity first
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const float m = bf<float>(h, b, s, NB_M);
    const float vx = nb_step_v(bf<float>(h, b, s, NB_VX), bf<float>(h, b, s, NB_FX), m, a.dt);
    const float vy = nb_step_v(bf<float>(h, b, s, NB_VY), bf<float>(h, b, s, NB_FY), m, a.dt);
    bf<float>(h, b, s, NB_VX) = vx;
    bf<float>(h, b, s, NB_VY) = vy;
    bf<float>(h, b, s, NB_X) = nb_step_p(bf<float>(h, b, s, NB_X), vx, a.dt);
    bf<float>(h, b, s, NB_Y) = nb_step_p(bf<float>(h, b, s, NB_Y), vy, a.dt);
    bf<uint32_t>(h, b, s, NB_TARGET) = kNone;
    bf<uint32_t>(h, b, s, NB_INCOMING) = kNone;
    bf<uint8_t>(h, b, s, NB_MERGED) = 0;
  }
};

// prepare_merge partials: per (i, chunk) the best (d2, j) with (m_j, j) >lex (m_i, i), d2 < R^2
// Merge search: for each body the nearest heavier (m, id) body within R, over
// the live list (an empty id is never a candidate: the exact test wants
// m_j > 0).  The common path of a tile entry is the packed distance and a
// running min; only a group of kMergeGroup entries that has some distance
// below the thread's largest current bound is re-examined with the exact
// per-body test (in ascending j, so ties resolve as in a sequential scan).
constexpr int kMergeGroup = 4;
__global__ void __launch_bounds__(kPairThreads) k_nb_merge_part(dsr_nbody_args a) {
  __shared__ float4 tile[256];
  const uint32_t nl = a.id_hi - a.id_lo;
  const PairI I(a);
  if (I.empty()) return;
  const float R2 = a.R * a.R;
  f32x2 PX[kNbPairs], PY[kNbPairs];
  float M[2 * kNbPairs], D[2 * kNbPairs];
  uint32_t B[2 * kNbPairs], ID[2 * kNbPairs];
#pragma unroll
  for (int q = 0; q < kNbPairs; ++q) {
    const float4 p0 = I.body(a, 2 * q, ID[2 * q]), p1 = I.body(a, 2 * q + 1, ID[2 * q + 1]);
    PX[q] = pk2(p0.x, p1.x);
    PY[q] = pk2(p0.y, p1.y);
    M[2 * q] = p0.z;
    M[2 * q + 1] = p1.z;
    // strict d2 < R^2, ties -> smaller j (j ascends); no body: bound -1 (searches nothing)
    D[2 * q] = ID[2 * q] != 0xFFFFFFFFu ? R2 : -1.f;
    D[2 * q + 1] = ID[2 * q + 1] != 0xFFFFFFFFu ? R2 : -1.f;
    B[2 * q] = B[2 * q + 1] = kNone;
  }
  float dmax = D[0];                                 // max of the D[] (they only decrease)
#pragma unroll
  for (int m = 1; m < 2 * kNbPairs; ++m) dmax = fmaxf(dmax, D[m]);
  const uint32_t jc = blockIdx.y, nj = live_n(a)[jc];
  const float4* J = live_s(a) + (size_t)jc * kChunk;
  for (uint32_t j0 = 0; j0 < nj; j0 += 256) {
    __syncthreads();
    const uint32_t ja = j0 + threadIdx.x, jb = ja + 128;
    // padding beyond the chunk's live bodies: far away, m = 0 (never a candidate)
    tile[threadIdx.x] = ja < nj ? __ldg(J + ja) : make_float4(1e18f, 1e18f, 0.f, 0.f);
    tile[threadIdx.x + 128] = jb < nj ? __ldg(J + jb) : make_float4(1e18f, 1e18f, 0.f, 0.f);
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < 256; k0 += kMergeGroup) {
      // per body (packed f32x2): e = dx^2 + dy^2 as fma(dx, dx, dy * dy)
      f32x2 E[kMergeGroup][kNbPairs];
      float emin = dmax;
#pragma unroll
      for (int g = 0; g < kMergeGroup; ++g) {
        const float4 p = tile[k0 + g];
        const f32x2 JX = pk2(p.x, p.x), JY = pk2(p.y, p.y);
#pragma unroll
        for (int q = 0; q < kNbPairs; ++q) {
          const f32x2 DX = sub2(JX, PX[q]), DY = sub2(JY, PY[q]);
          E[g][q] = fma2(DX, DX, mul2(DY, DY));
          float e0, e1;
          upk2(E[g][q], e0, e1);
          emin = fminf(emin, fminf(e0, e1));
        }
      }
      if (emin < dmax) {                             // rare: some body within its bound
#pragma unroll
        for (int g = 0; g < kMergeGroup; ++g) {
          const float4 p = tile[k0 + g];
          const uint32_t j = __float_as_uint(p.w);
#pragma unroll
          for (int q = 0; q < kNbPairs; ++q) {
            float e[2];
            upk2(E[g][q], e[0], e[1]);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t i = ID[2 * q + u];
              const float mi = M[2 * q + u];
              if (e[u] < D[2 * q + u] && p.z > 0.f && (p.z > mi || (p.z == mi && j > i))) {
                D[2 * q + u] = e[u];
                B[2 * q + u] = j;
              }
            }
          }
        }
        dmax = D[0];
#pragma unroll
        for (int m = 1; m < 2 * kNbPairs; ++m) dmax = fmaxf(dmax, D[m]);
      }
    }
  }
  uint2* part = reinterpret_cast<uint2*>(a.scratch) + (size_t)blockIdx.y * nl;
#pragma unroll
  for (int m = 0; m < 2 * kNbPairs; ++m)
    if (ID[m] != 0xFFFFFFFFu) part[ID[m] - a.id_lo] = make_uint2(__float_as_uint(D[m]), B[m]);
}

__global__ void k_nb_merge_pick(DevHeap h, dsr_nbody_args a) {
  const uint32_t nl = a.id_hi - a.id_lo, chunks = (a.n_total + kChunk - 1) / kChunk;
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < nl; li += gridDim.x * blockDim.x) {
    const uint32_t i = a.id_lo + li;
    const uint64_t hd = a.shandle[i];
    if (!hd) continue;
    uint32_t best = kNone;
    float bd = 0.f;
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint2 v = reinterpret_cast<const uint2*>(a.scratch)[(size_t)c * nl + li];
      const float d = __uint_as_float(v.x);
      if (v.y != kNone && (best == kNone || d < bd)) { best = v.y; bd = d; }   // chunks ascend in j
    }
    a.target[i] = best;
    bf<uint32_t>(h, h_bid(hd), h_slot(hd), NB_TARGET) = best;
  }
}

// claim over all ids: at most one absorption per target per step, smallest id wins
__global__ void k_nb_claim_all(uint64_t n, dsr_nbody_args a) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = a.target[i];
    if (t != kNone) atomicMin(a.incoming + t, (uint32_t)i);
  }
}
struct NbClaim {  // do-all form of the claim (single GPU): incoming[target] = min id
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t t = bf<uint32_t>(h, b, s, NB_TARGET);
    if (t != kNone) atomicMin(a.incoming + t, bf<uint32_t>(h, b, s, NB_ID));
  }
};

struct NbAbsorb { // perfectly inelastic merge: momentum and centre of mass
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t id = bf<uint32_t>(h, b, s, NB_ID);
    const uint32_t i = a.incoming[id];
    bf<uint32_t>(h, b, s, NB_INCOMING) = i;
    if (i == kNone || a.target[id] != kNone) return;
    const float4 pi = s4(a, i);
    const float2 vi = reinterpret_cast<const float2*>(a.V)[i];
    const float m = bf<float>(h, b, s, NB_M), mi = pi.z;
    const float mn = __fadd_rn(m, mi);
    bf<float>(h, b, s, NB_VX) = nb_mix(m, bf<float>(h, b, s, NB_VX), mi, vi.x, mn);
    bf<float>(h, b, s, NB_VY) = nb_mix(m, bf<float>(h, b, s, NB_VY), mi, vi.y, mn);
    bf<float>(h, b, s, NB_X) = nb_mix(m, bf<float>(h, b, s, NB_X), mi, pi.x, mn);
    bf<float>(h, b, s, NB_Y) = nb_mix(m, bf<float>(h, b, s, NB_Y), mi, pi.y, mn);
    bf<float>(h, b, s, NB_M) = mn;
  }
};

struct NbDeleteMerged {   // step_6_delete_merged: merged iff my claim won an absorbing target
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t id = bf<uint32_t>(h, b, s, NB_ID);
    const uint32_t t = a.target[id];
    const bool merged = t != kNone && a.incoming[t] == id && a.target[t] == kNone;
    bf<uint8_t>(h, b, s, NB_MERGED) = merged;
    if (merged) dsr_destroy(h, make_handle(0, h.types[0].cap, b, s));
  }
};

struct NbDump {
  typedef dsr_nbody_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t, uint32_t b, uint32_t s, const Args& a, Acc&) {
    float* o = a.out + 6ull * bf<uint32_t>(h, b, s, NB_ID);
    o[0] = bf<float>(h, b, s, NB_X);
    o[1] = bf<float>(h, b, s, NB_Y);
    o[2] = bf<float>(h, b, s, NB_VX);
    o[3] = bf<float>(h, b, s, NB_VY);
    o[4] = bf<float>(h, b, s, NB_M);
    o[5] = 1.f;
  }
};

bool nb_method_info(uint32_t id, MethodInfo* mi) {
  if (id >= DSR_M_NB_SNAPSHOT && id <= DSR_M_NB_DUMP) {
    *mi = {id == DSR_M_NB_DELETE_MERGED ? 1 : 0, sizeof(dsr_nbody_args)};   // delete_merged self-deletes
    return true;
  }
  return false;
}

// peer mode: the launching stream waits (front end, no SM held) until every
// other rank's flag slot slot0 + r reached epoch + 1
static bool peer_wait(const dsr_nbody_args& a, uint32_t slot0, cudaStream_t st) {
  if (!a.npeers) return true;
  typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn wait = nullptr;
  if (!wait) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    wait = (WaitFn)fn;
  }
  for (uint32_t r = 0; r < a.world; ++r)
    if (r != a.rank && wait((CUstream)st, (CUdeviceptr)(a.flags + slot0 + r), a.epoch + 1u, CU_STREAM_WAIT_VALUE_GEQ) !=
                           CUDA_SUCCESS)
      return false;
  return true;
}

// x: the i-blocks of the live-list chunks that hold my ids; y: the j chunks
static dim3 pair_grid(const dsr_nbody_args& a) {
  return dim3(((a.id_hi - 1) / kChunk - a.id_lo / kChunk + 1) * kIBlocksPerChunk, (a.n_total + kChunk - 1) / kChunk);
}
static void launch_live(const dsr_nbody_args& a, cudaStream_t st) {
  k_nb_live<<<(a.n_total + kChunk - 1) / kChunk, kLiveThreads, 0, st>>>(a);
}

bool nb_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  const dsr_nbody_args& a = *(const dsr_nbody_args*)args;
  switch (id) {
    case DSR_M_NB_SNAPSHOT: launch_doall<NbSnapshot>(c, T, snapshot, args); return true;
    case DSR_M_NB_FORCE:
      if (a.id_hi <= a.id_lo || !a.live) return a.id_hi <= a.id_lo;
      if (!peer_wait(a, 0, c.st)) return false;
      launch_live(a, c.st);
      k_nb_force_part<<<pair_grid(a), kPairThreads, 0, c.st>>>(a);
      k_nb_force_sum<<<grid_for(c, a.id_hi - a.id_lo, k_nb_force_sum), 256, 0, c.st>>>(c.h, a);
      count_launch(3);
      return true;
    case DSR_M_NB_MOVE: launch_doall<NbMove>(c, T, snapshot, args); return true;
    case DSR_M_NB_PREPARE_MERGE:
      if (a.id_hi <= a.id_lo || !a.live) return a.id_hi <= a.id_lo;
      if (!peer_wait(a, 0, c.st)) return false;
      launch_live(a, c.st);
      k_nb_merge_part<<<pair_grid(a), kPairThreads, 0, c.st>>>(a);
      k_nb_merge_pick<<<grid_for(c, a.id_hi - a.id_lo, k_nb_merge_pick), 256, 0, c.st>>>(c.h, a);
      count_launch(3);
      return true;
    case DSR_M_NB_CLAIM: launch_doall<NbClaim>(c, T, snapshot, args); return true;
    case DSR_M_NB_ABSORB: launch_doall<NbAbsorb>(c, T, snapshot, args); return true;
    case DSR_M_NB_DELETE_MERGED: launch_doall<NbDeleteMerged>(c, T, snapshot, args); return true;
    case DSR_M_NB_DUMP: launch_doall<NbDump>(c, T, snapshot, args); return true;
  }
  return false;
}

bool nb_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_K_NB_CLEAR_SNAPSHOT && id != DSR_K_NB_CLAIM && id != DSR_K_NB_SIGNAL && id != DSR_K_NB_PUSH_TARGET)
    return false;
  if (bytes != sizeof(dsr_nbody_args)) { *ok = 0; return true; }
  const dsr_nbody_args a = *(const dsr_nbody_args*)args;
  if (n != a.n_total || a.npeers > 7 || (a.npeers && (!a.flags || a.world != a.npeers + 1 || a.rank >= a.world))) {
    *ok = 0;
    return true;
  }
  if ((id == DSR_K_NB_SIGNAL || id == DSR_K_NB_PUSH_TARGET) && !a.npeers) { *ok = 0; return true; }
  if (id == DSR_K_NB_CLEAR_SNAPSHOT) {
    k_nb_clear<<<grid_for(c, n, k_nb_clear), 256, 0, c.st>>>(n, a);
  } else if (id == DSR_K_NB_CLAIM) {
    if (!peer_wait(a, a.world, c.st)) { *ok = 0; return true; }
    k_nb_claim_all<<<grid_for(c, n, k_nb_claim_all), 256, 0, c.st>>>(n, a);
  } else if (id == DSR_K_NB_SIGNAL) {
    k_nb_signal<<<1, 32, 0, c.st>>>(a, 0);
  } else {
    k_nb_push_target<<<grid_for(c, a.id_hi - a.id_lo, k_nb_push_target), 256, 0, c.st>>>(a);
    k_nb_signal<<<1, 32, 0, c.st>>>(a, a.world);
    count_launch();
  }
  count_launch();
  return true;
}

bool nb_ctor_launch(uint32_t id, const LaunchCtx& c, uint32_t T, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_C_NB_BODY) return false;
  if (bytes != sizeof(dsr_nbody_args) || T != 0) { *ok = 0; return true; }
  const dsr_nbody_args a = *(const dsr_nbody_args*)args;
  if (n != (uint64_t)(a.id_hi - a.id_lo) || a.id_hi > a.n_total) { *ok = 0; return true; }
  k_nb_new<<<grid_for(c, n, k_nb_new), 256, 0, c.st>>>(c.h, n, a);
  count_launch();
  return true;
}

// ---- static-allocation baseline: the same
// six passes on id-indexed SOA arrays (S = (x, y, m, 0), V = (vx, vy); a dead
// id has m = 0), no heap, no objects.  The all-pairs kernels are the ones
// above (they read S only); the per-body passes are array loops with the
// operations and order of NbMove / k_nb_merge_pick / NbAbsorb /
// NbDeleteMerged, so a run equals the heap version bit for bit.
__global__ void k_nbs_force_move(dsr_nbody_args a) {
  const uint32_t n = a.n_total, chunks = (n + kChunk - 1) / kChunk;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    a.target[i] = kNone;
    a.incoming[i] = kNone;
    float4 p = reinterpret_cast<float4*>(a.S)[i];
    if (p.z == 0.f) continue;                                     // dead id
    float ax = 0.f, ay = 0.f;
    for (uint32_t c = 0; c < chunks; ++c) {
      const float2 v = reinterpret_cast<const float2*>(a.scratch)[(size_t)c * n + i];
      ax += v.x;
      ay += v.y;
    }
    const float gm = __fmul_rn(a.G, p.z);
    const float fx = __fmul_rn(gm, ax), fy = __fmul_rn(gm, ay);
    float2 v = reinterpret_cast<float2*>(a.V)[i];
    v.x = nb_step_v(v.x, fx, p.z, a.dt);
    v.y = nb_step_v(v.y, fy, p.z, a.dt);
    p.x = nb_step_p(p.x, v.x, a.dt);
    p.y = nb_step_p(p.y, v.y, a.dt);
    reinterpret_cast<float2*>(a.V)[i] = v;
    reinterpret_cast<float4*>(a.S)[i] = p;
  }
}
__global__ void k_nbs_merge_pick(dsr_nbody_args a) {
  const uint32_t n = a.n_total, chunks = (n + kChunk - 1) / kChunk;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (reinterpret_cast<const float4*>(a.S)[i].z == 0.f) continue;
    uint32_t best = kNone;
    float bd = 0.f;
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint2 v = reinterpret_cast<const uint2*>(a.scratch)[(size_t)c * n + i];
      const float d = __uint_as_float(v.x);
      if (v.y != kNone && (best == kNone || d < bd)) { best = v.y; bd = d; }
    }
    a.target[i] = best;
  }
}
__global__ void k_nbs_absorb(dsr_nbody_args a) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < a.n_total; id += gridDim.x * blockDim.x) {
    const uint32_t i = a.incoming[id];
    if (i == kNone || a.target[id] != kNone) continue;
    float4 p = reinterpret_cast<float4*>(a.S)[id];
    float2 v = reinterpret_cast<float2*>(a.V)[id];
    const float4 pi = reinterpret_cast<const float4*>(a.S)[i];     // i merges away: nobody writes it here
    const float2 vi = reinterpret_cast<const float2*>(a.V)[i];
    const float m = p.z, mi = pi.z, mn = __fadd_rn(m, mi);
    v.x = nb_mix(m, v.x, mi, vi.x, mn);
    v.y = nb_mix(m, v.y, mi, vi.y, mn);
    p.x = nb_mix(m, p.x, mi, pi.x, mn);
    p.y = nb_mix(m, p.y, mi, pi.y, mn);
    p.z = mn;
    reinterpret_cast<float2*>(a.V)[id] = v;
    reinterpret_cast<float4*>(a.S)[id] = p;
  }
}
__global__ void k_nbs_delete(dsr_nbody_args a) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < a.n_total; id += gridDim.x * blockDim.x) {
    const uint32_t t = a.target[id];
    if (t != kNone && a.incoming[t] == id && a.target[t] == kNone) reinterpret_cast<float4*>(a.S)[id].z = 0.f;
  }
}

}  // namespace dsr

extern "C" dsr_status dsr_nbody_static_step(const dsr_nbody_static_args* sa, uint32_t steps, void* stream) {
  using namespace dsr;
  if (!sa || !sa->S || !sa->V || !sa->target || !sa->incoming || !sa->scratch || !sa->live || sa->n == 0)
    return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  dsr_nbody_args a;
  memset(&a, 0, sizeof(a));
  a.S = sa->S;
  a.V = sa->V;
  a.target = sa->target;
  a.incoming = sa->incoming;
  a.scratch = sa->scratch;
  a.live = sa->live;
  a.G = sa->G; a.dt = sa->dt; a.eps = sa->eps; a.R = sa->R;
  a.n_total = sa->n;
  a.id_lo = 0;
  a.id_hi = sa->n;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return DSR_ERR_CUDA;
  const int g = (int)std::min<uint64_t>((sa->n + 255) / 256, (uint64_t)sms * 8);
  for (uint32_t k = 0; k < steps; ++k) {
    launch_live(a, st);
    k_nb_force_part<<<pair_grid(a), kPairThreads, 0, st>>>(a);           // compute_force over S0
    k_nbs_force_move<<<g, 256, 0, st>>>(a);                             // + move: S becomes S1
    if (sa->merges) {
      launch_live(a, st);
      k_nb_merge_part<<<pair_grid(a), kPairThreads, 0, st>>>(a);        // prepare_merge over S1
      k_nbs_merge_pick<<<g, 256, 0, st>>>(a);
      k_nb_claim_all<<<g, 256, 0, st>>>(a.n_total, a);
      k_nbs_absorb<<<g, 256, 0, st>>>(a);
      k_nbs_delete<<<g, 256, 0, st>>>(a);
      count_launch(6);
    }
    count_launch(3);
  }
  return cudaGetLastError() == cudaSuccess ? DSR_OK : DSR_ERR_CUDA;
}
