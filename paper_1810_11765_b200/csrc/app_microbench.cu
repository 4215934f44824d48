// app_microbench.cu -- allocator microbenchmark (BASELINE configs[4], SURVEY
// c.4), Linux Scalability and the allocator test kernels
// (single-thread replay, concurrent torture, handle collection).
#include "dsr_host.h"
#include "dsr_doall.cuh"

namespace dsr {

__constant__ uint32_t kMbType[4] = {0, 0, 1, 2};
#ifndef DSR_MB_CHUNK
#define DSR_MB_CHUNK 2
#endif
#ifndef DSR_MB_FREEODD_SNAP
#define DSR_MB_FREEODD_SNAP 1
#endif
#ifndef DSR_MB_MINB
#define DSR_MB_MINB 8
#endif
constexpr uint32_t kMbChunk = DSR_MB_CHUNK;   // warp work unit: 2 x 32 consecutive t (sweeps: 2/4/8/16)

// ---- phase 1 / 4: user kernel, thread t does new [A,A,B,C][t&3] (device new)
// (MINB CTAs x 256 threads per SM; latency-bound, so occupancy matters).  The
// CTA-coalescing ablation (DSR_F_CTA_NEW) is a separate instantiation so the
// default kernel carries none of its 16 KB of shared memory.
// IN: the field values come from the caller's array a.in (end-to-end runs with
// host-resident inputs) instead of being computed from the key.
template <bool CTA, int MINB, bool IN = false>
__global__ void __launch_bounds__(256, MINB) k_mb_new(DevHeap h, uint64_t n, dsr_mb_new_args a) {
  const uint64_t kp = rng_prefix(a.seed, 0);
  auto one = [&](uint64_t i, uint64_t hd) {
    if (!hd) return;
    const uint64_t t = a.t0 + i;
    const uint32_t T = h_type(hd);
    const uint32_t nf = h.types[T].nfields;
    // the object's slot in column 0; column k is col_off[k] bytes further (u32 fields)
    uint8_t* const obj = h.data + (size_t)h_bid(hd) * h.block_bytes + 4u * h_slot(hd);
    const uint32_t* src = IN ? a.in + 16 * (i >> 2) + ((0xA630u >> (4 * (i & 3))) & 0xFu) : nullptr;
    for (uint32_t k = 0; k < nf; ++k)
      *reinterpret_cast<uint32_t*>(obj + h.types[T].col_off[k]) = IN ? __ldg(src + k) : (uint32_t)rng_key_p(kp, 5, t * 16 + k);
  };
  if (CTA) {
    // uniform trip count: every thread of the CTA reaches dsr_new_uniform together
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
      const uint64_t i = base + threadIdx.x;
      one(i, dsr_new_uniform(h, kMbType[(a.t0 + i) & 3], i < n));
    }
    return;
  }
  // Dynamic work distribution: a warp takes the next kMbChunk x 32 threads'
  // worth of t from a device counter, so warps slowed by allocation contention
  // do not leave a tail of idle SMs (static striding left half the warps idle
  // on average, ncu achieved occupancy 49 %).
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&h.ctrl[CTRL_WORK], 32ull * kMbChunk);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    for (uint32_t k = 0; k < kMbChunk; ++k) {
      const uint64_t i = base + 32ull * k + lane;
      const uint32_t r = (uint32_t)((a.t0 + i) & 3);
      one(i, i < n ? dsr_new(h, r ? r - 1 : 0) : 0ull);                  // [A, A, B, C][t & 3]
    }
  }
}

// ---- phase 1 / 4, batched: the same objects (thread t -> [A,A,B,C][t&3],
// field k = low32(key(seed, 0, MB_FIELD, 16t + k))), but each warp takes a
// work unit of kMbUnit consecutive t and allocates all objects of one type
// of the unit with ONE warp-cooperative request (dsr_new_warp, reading
// R-BULK) instead of one coalesced request per 32 threads; the constructor
// then writes the reserved slots chunk by chunk (lane j -> slot j of a chunk:
// coalesced column stores).  3072 t = 1536 A + 768 B + 768 C = exactly 24 / 16 / 24
// blocks of N_T = 64 / 48 / 32.
#ifndef DSR_MB_UNIT
#define DSR_MB_UNIT 3072
#endif
constexpr uint32_t kMbUnit = DSR_MB_UNIT;

// Constructor of the reserved slots of one dsr_new_warp call for type T.
// The objects are ranked in lane order of the chunks, then by slot: the chunk
// of lane c holds objects done + cum_c ...
//  * quads: a chunk that is one run of slots starting at a multiple of 4
//    (every fresh block, the free tail of a block) is cut into quads of 4
//    slots; the warp's quads of all such chunks are dealt out to the lanes (a
//    per-warp table in shared memory, walked with a cursor), and a lane
//    computes the 4 objects' keys and writes each column with one 128-bit
//    store; the last cnt % 4 objects of such a chunk are written by the lane
//    that holds the chunk;
//  * other chunks (holes of partly freed blocks): chunk by chunk, lane j ->
//    the chunk's j-th reserved slot, looked up in a per-warp slot list the
//    lanes build with one popc each (no per-object n-th-bit search).
// One copy of each loop for all types, with the field loop not unrolled and
// the column offsets read from the kernel parameter space: the constructor's
// instruction footprint, not its instruction count, decided its speed (ncu:
// "no instruction" was the top stall with an unrolled copy per type).
// sw: this warp's shared scratch, kMbScratch words.
constexpr uint32_t kMbScratch = 4 * 32 + 16;
#ifndef DSR_MB_KEYMAD
#define DSR_MB_KEYMAD 1
#endif
#ifndef DSR_MB_KEYHI
#define DSR_MB_KEYHI 1
#endif
// 1, but not a constant to the compiler: multiplies by it (and by its powers
// of two) stay IMADs on the FMA pipe instead of being folded into adds and
// shifts on the ALU pipe (pipe balancing of the key's mix, see sm64_mix_lo)
__constant__ uint32_t kMbOne = 1;
// low 32 bits of sm64 after its first step (z = x + G).  The key is 11 ALU-pipe
// instructions (shifts, xors) to 9 FMA-pipe ones (the 64-bit multiplies); each
// pipe takes a warp instruction every 2 cycles per scheduler, so with KEYHI the
// high word's first shift (hi >> 30) is a multiply-high by 4 (= one << 2).
__device__ __forceinline__ uint32_t sm64_mix_lo(uint64_t z, uint32_t one) {
#if DSR_MB_KEYHI
  const uint32_t hi = (uint32_t)(z >> 32), lo = (uint32_t)z;
  z = ((uint64_t)(hi ^ __umulhi(hi, one << 2)) << 32 | (lo ^ (uint32_t)(z >> 30))) * 0xBF58476D1CE4E5B9ull;
#else
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
#endif
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z ^ (z >> 31));
}
// t of the i-th object of type T in the unit (residues off0 [, off1] of t & 3)
__device__ __forceinline__ uint64_t mb_t(uint64_t ts, uint32_t nres, uint32_t off0, uint32_t off1, uint32_t i) {
  return nres == 2 ? ts + 4ull * (i >> 1) + ((i & 1) ? off1 : off0) : ts + 4ull * i + off0;
}
// the same for 4 independent keys, step by step (the 4 dependent chains
// interleaved in program order, so a warp has 4 independent instructions to
// issue back to back instead of waiting out each one's latency)
#ifndef DSR_MB_KEY4
#define DSR_MB_KEY4 1
#endif
__device__ __forceinline__ void sm64_mix_lo4(uint64_t z[4], uint32_t one, uint32_t v[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#if DSR_MB_KEYHI
    const uint32_t hi = (uint32_t)(z[j] >> 32), lo = (uint32_t)z[j];
    z[j] = (uint64_t)(hi ^ __umulhi(hi, one << 2)) << 32 | (lo ^ (uint32_t)(z[j] >> 30));
#else
    z[j] ^= z[j] >> 30;
#endif
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) z[j] *= 0xBF58476D1CE4E5B9ull;
#pragma unroll
  for (int j = 0; j < 4; ++j) z[j] ^= z[j] >> 27;
#pragma unroll
  for (int j = 0; j < 4; ++j) z[j] *= 0x94D049BB133111EBull;
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = (uint32_t)(z[j] ^ (z[j] >> 31));
}
template <bool IN>
__device__ __forceinline__ void mb_construct(const DevHeap& h, uint32_t T, const dsr_mb_new_args& a, uint64_t kp,
                                             uint64_t ts, uint32_t nres, uint32_t off0, uint32_t off1, uint32_t done,
                                             uint32_t bid, uint64_t mask, uint32_t* sw) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nf = h.types[T].nfields;
  const uint32_t cnt = (uint32_t)__popcll(mask);
  uint32_t cum = cnt;                                      // exclusive prefix in lane order
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, cum, o);
    if (lane >= (uint32_t)o) cum += v;
  }
  cum -= cnt;
  // one object: slot s of block b, the i-th of T in the unit (fields unrolled
  // up to the microbench's largest type, column offsets in registers)
  constexpr uint32_t kMaxF = 6;
  uint32_t col[kMaxF];
#pragma unroll
  for (uint32_t k = 0; k < kMaxF; ++k) col[k] = k < nf ? h.types[T].col_off[k] : 0u;
  auto construct = [&](uint32_t b, uint32_t s, uint32_t i) {
#ifdef DSR_DEBUG
    if (b >= h.M || s >= h.types[T].cap) {
      atomicOr(&h.ctrl[CTRL_ERR], (unsigned long long)ERRB_BOUNDS);
      return;
    }
#endif
    const uint64_t t = mb_t(ts, nres, off0, off1, i);
    uint8_t* const obj = h.data + (size_t)b * h.block_bytes + 4u * s;
    const uint32_t* src = nullptr;
    if (IN) {
      const uint64_t ti = t - a.t0;
      src = a.in + 16 * (ti >> 2) + ((0xA630u >> (4 * (ti & 3))) & 0xFu);
    }
#pragma unroll
    for (uint32_t k = 0; k < kMaxF; ++k)
      if (k < nf) *reinterpret_cast<uint32_t*>(obj + col[k]) = IN ? __ldg(src + k) : (uint32_t)rng_key_p(kp, 5, t * 16 + k);
  };
  const uint32_t lo = mask ? ctz64(mask) : 0u;
  const uint64_t run = mask >> lo;
  const bool quad = !IN && mask != 0 && (lo & 3u) == 0 && (run & (run + 1ull)) == 0;
  const uint32_t nq = quad ? cnt >> 2 : 0u;                // full quads
  const uint32_t qball = __ballot_sync(0xffffffffu, nq != 0);
  if (qball) {
    uint32_t qin = nq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, qin, o);
      if (lane >= (uint32_t)o) qin += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, qin, 31);
    const uint32_t nqc = (uint32_t)__popc(qball);
    if (nq) {                                              // table entry: quad start, block, first slot, first object
      const uint32_t e = (uint32_t)__popc(qball & lt);
      sw[e] = qin - nq;
      sw[32 + e] = bid;
      sw[64 + e] = lo;
      sw[96 + e] = cum + done;
    }
    __syncwarp();
    const uint64_t kx = kp ^ (5ull << 40);                 // key of field k of t = sm64(kx ^ (16 t + k)), 16 t + k < 2^40
#if DSR_MB_KEYMAD
    // sm64 starts with x + G.  x = kx ^ 16t ^ k = (kx ^ 16t ^ c) + (c ^ k), c = kx & 15:
    // per object Y = (kx ^ 16t ^ c) + G, per field z = Y + (c ^ k) as one
    // IMAD.WIDE.U32 (c ^ k) * one + Y on the FMA pipe (the key's xor-shifts
    // keep the ALU pipe the busier one; `one` is 1 but not a constant to ptxas,
    // which would turn the multiply-add back into an IADD3 pair)
    const uint32_t cx = (uint32_t)kx & 15u;
    const uint32_t one = kMbOne;
#endif
    // the quad's chunk: when all quad chunks have the same length (whole fresh
    // blocks: the common case), g / nq by a float reciprocal (exact after one
    // upward correction for g < 2^20); otherwise a cursor over the table
    const uint32_t nqmax = __reduce_max_sync(0xffffffffu, nq);
    const bool even = __reduce_min_sync(0xffffffffu, nq ? nq : 0xFFFFFFFFu) == nqmax;
    const float rq = __frcp_rn((float)nqmax);
    // t of the 4 objects of a quad from the first one's: t0 + {0, u, w, u + w}
    // (nres = 1: u = 4, w = 8; nres = 2: w = 4, u = off1 - off0 if the first
    // object has residue off0, else 4 - (off1 - off0))
    const uint32_t w = nres == 2 ? 4u : 8u;
    uint32_t cur = 0;
    for (uint32_t g = lane; g < total; g += 32) {
      uint32_t q;
      if (even) {
        cur = (uint32_t)((float)g * rq);
        q = g - cur * nqmax;
        if (q >= nqmax) { q -= nqmax; ++cur; }
      } else {
        while (cur + 1 < nqc && sw[cur + 1] <= g) ++cur;
        q = g - sw[cur];
      }
      const uint32_t i = sw[96 + cur] + 4u * q;
#ifdef DSR_DEBUG
      // the quad lies in its chunk's run of reserved slots, inside the block
      if (cur >= nqc || sw[32 + cur] >= h.M || sw[64 + cur] + 4u * q + 4u > h.types[T].cap ||
          q >= (cur + 1 < nqc ? sw[cur + 1] : total) - sw[cur]) {
        atomicOr(&h.ctrl[CTRL_ERR], (unsigned long long)ERRB_BOUNDS);
        continue;
      }
#endif
      uint8_t* const p = h.data + (size_t)sw[32 + cur] * h.block_bytes + 4u * (sw[64 + cur] + 4u * q);
      const uint64_t t0 = mb_t(ts, nres, off0, off1, i);
      const uint32_t u = nres == 2 ? ((i & 1) ? 4u - (off1 - off0) : off1 - off0) : 4u;
      const uint64_t x0 = kx ^ (t0 << 4), x1 = kx ^ ((t0 + u) << 4);
      const uint64_t x2 = kx ^ ((t0 + w) << 4), x3 = kx ^ ((t0 + u + w) << 4);
#if DSR_MB_KEYMAD
      const uint64_t y0 = (x0 ^ cx) + 0x9E3779B97F4A7C15ull, y1 = (x1 ^ cx) + 0x9E3779B97F4A7C15ull;
      const uint64_t y2 = (x2 ^ cx) + 0x9E3779B97F4A7C15ull, y3 = (x3 ^ cx) + 0x9E3779B97F4A7C15ull;
#endif
#pragma unroll 1
      for (uint32_t k = 0; k < nf; ++k) {
#if DSR_MB_KEYMAD && DSR_MB_KEY4
        const uint32_t ck = cx ^ k;
        uint64_t z[4] = {y0 + (uint64_t)ck * one, y1 + (uint64_t)ck * one, y2 + (uint64_t)ck * one, y3 + (uint64_t)ck * one};
        uint32_t v[4];
        sm64_mix_lo4(z, one, v);
        const uint32_t v0 = v[0], v1 = v[1], v2 = v[2], v3 = v[3];
#elif DSR_MB_KEYMAD
        const uint32_t ck = cx ^ k;
        const uint32_t v0 = sm64_mix_lo(y0 + (uint64_t)ck * one, one), v1 = sm64_mix_lo(y1 + (uint64_t)ck * one, one);
        const uint32_t v2 = sm64_mix_lo(y2 + (uint64_t)ck * one, one), v3 = sm64_mix_lo(y3 + (uint64_t)ck * one, one);
#else
        const uint32_t v0 = (uint32_t)sm64(x0 ^ (uint64_t)k), v1 = (uint32_t)sm64(x1 ^ (uint64_t)k);
        const uint32_t v2 = (uint32_t)sm64(x2 ^ (uint64_t)k), v3 = (uint32_t)sm64(x3 ^ (uint64_t)k);
#endif
        *reinterpret_cast<uint4*>(p + h.types[T].col_off[k]) = make_uint4(v0, v1, v2, v3);
      }
    }
    __syncwarp();
  }
  // the last cnt % 4 objects of a quad chunk: by the lane that holds it
  if (quad)
    for (uint32_t j = 4u * nq; j < cnt; ++j) construct(bid, lo + j, cum + done + j);
  uint32_t chunks = __ballot_sync(0xffffffffu, mask != 0 && !quad);
  uint8_t* const slots = reinterpret_cast<uint8_t*>(sw + 128);
  while (chunks) {
    const uint32_t c = __ffs(chunks) - 1;
    chunks &= chunks - 1;
    const uint32_t cb = __shfl_sync(0xffffffffu, bid, c);
    const uint64_t cm = shfl64(0xffffffffu, mask, c);
    const uint32_t c0 = __shfl_sync(0xffffffffu, cum, c) + done;
    const uint32_t cn = (uint32_t)__popcll(cm);
    // slot list: lane p places slots p and p + 32 at their ranks
    const uint32_t mlo = (uint32_t)cm, mhi = (uint32_t)(cm >> 32);
    if ((mlo >> lane) & 1u) slots[__popc(mlo & lt)] = (uint8_t)lane;
    if ((mhi >> lane) & 1u) slots[__popc(mlo) + __popc(mhi & lt)] = (uint8_t)(lane + 32);
    __syncwarp();
#ifdef DSR_DEBUG
    for (uint32_t j = lane; j < cn; j += 32)
      if (!((cm >> slots[j]) & 1ull)) atomicOr(&h.ctrl[CTRL_ERR], (unsigned long long)ERRB_BOUNDS);   // not reserved
#endif
    for (uint32_t j = lane; j < cn; j += 32) construct(cb, slots[j], c0 + j);
    __syncwarp();
  }
}

#ifndef DSR_MB_BULK_MINB
#define DSR_MB_BULK_MINB 4   // CTAs x 256 threads per SM (64 registers, no spills); see DESIGN §6 for the sweep
#endif
template <bool IN = false>
__global__ void __launch_bounds__(256, DSR_MB_BULK_MINB) k_mb_new_bulk(DevHeap h, uint64_t n, dsr_mb_new_args a) {
  const uint64_t kp = rng_prefix(a.seed, 0);
  const uint32_t lane = threadIdx.x & 31;
  __shared__ uint32_t s_scr[8][kMbScratch];
  uint32_t* const sw = s_scr[threadIdx.x >> 5];
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&h.ctrl[CTRL_WORK], (unsigned long long)kMbUnit);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    const uint32_t un = (uint32_t)(n - base < kMbUnit ? n - base : kMbUnit);
    const uint64_t ts = a.t0 + base;                       // first t of the unit
#pragma unroll 1
    for (uint32_t T = 0; T < 3; ++T) {
      // residues r = t & 3 of type T ([A,A,B,C]) as offsets from ts, ascending
      uint32_t off0 = 0, off1 = 0, nres = 0;
#pragma unroll
      for (uint32_t d = 0; d < 4; ++d) {
        const uint32_t r = (uint32_t)((ts + d) & 3);
        if ((r ? r - 1 : 0) == T) {
          if (nres == 0) off0 = d; else off1 = d;
          ++nres;
        }
      }
      // objects of T among ts .. ts + un - 1
      uint32_t need = off0 < un ? (un - off0 + 3) / 4 : 0;
      if (nres == 2) need += off1 < un ? (un - off1 + 3) / 4 : 0;
      uint32_t done = 0;
      while (done < need) {
        uint32_t bid;
        uint64_t mask;
        const uint32_t got = dsr_new_warp(h, T, need - done, &bid, &mask);
        if (!got) break;                                   // OOM (sticky error set)
        mb_construct<IN>(h, T, a, kp, ts, nres, off0, off1, done, bid, mask, sw);
        done += got;
      }
    }
  }
}

// ---- phase 2 / 5: field reduction.  Vectorised do-all body: one thread per
// 4 consecutive slots ("quad") of a block; each field column is read with one
// 128-bit non-coherent load per quad (16 lanes cover a 64-slot u32 column).
template <int NF>
__global__ void __launch_bounds__(256) k_mb_reduce(DevHeap h, uint32_t T, unsigned long long* out3) {
  const uint32_t r = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RCOUNT]);
  const uint32_t Q = h.types[T].cap >> 2;         // caps 64/48/32 are multiples of 4
  const uint64_t total = (uint64_t)r * Q;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t cols[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) cols[f] = h.types[T].col_off[f];
  uint64_t cnt = 0, sum = 0;
  uint32_t x = 0;
  // quad e -> (block index, quad) = (e / Q, e % Q), advanced incrementally by the grid stride
  uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t bi = e / Q;
  uint32_t q = (uint32_t)(e - bi * Q);
  const uint64_t dbi = stride / Q;
  const uint32_t dq = (uint32_t)(stride - dbi * Q);
  for (; e < total; e += stride, bi += dbi, q += dq) {
    if (q >= Q) { q -= Q; ++bi; }
    const uint32_t b = __ldg(h.R + bi);
    const uint32_t m4 = (uint32_t)(__ldg((const unsigned long long*)h.alloc_bm + b) >> (4 * q)) & 0xFu;
    if (!m4) continue;
    const uint8_t* base = h.data + (size_t)b * h.block_bytes + 16u * q;
    uint4 v[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) v[f] = __ldcs(reinterpret_cast<const uint4*>(base + cols[f]));
    cnt += __popc(m4);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const uint32_t a0 = (m4 & 1) ? v[f].x : 0u, a1 = (m4 & 2) ? v[f].y : 0u;
      const uint32_t a2 = (m4 & 4) ? v[f].z : 0u, a3 = (m4 & 8) ? v[f].w : 0u;
      sum += (uint64_t)a0 + a1 + (uint64_t)a2 + a3;
      x ^= a0 ^ a1 ^ a2 ^ a3;
    }
  }
  // warp then CTA reduction, one atomic per CTA and output
  __shared__ unsigned long long s_c[8], s_s[8];
  __shared__ uint32_t s_x[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    x ^= __shfl_xor_sync(0xffffffffu, x, o);
  }
  const uint32_t wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_c[wid] = cnt; s_s[wid] = sum; s_x[wid] = x; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = 0, s = 0;
    uint32_t xx = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { c += s_c[k]; s += s_s[k]; xx ^= s_x[k]; }
    if (c) {
      atomicAdd(out3 + 0, c);
      atomicAdd(out3 + 1, s);
      atomicXor(out3 + 2, (unsigned long long)xx);
    }
  }
}

// ---- phase 3 / 6: self-deletion methods
struct MbFreeOdd {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args&, Acc&) {
    // read-only, and the destroy is control-dependent on the read: no release needed
    if (*field_ptr<uint32_t>(h, T, 0, b, s) & 1u) dsr_destroy_ro(h, make_handle(T, h.types[T].cap, b, s));
  }
};
struct MbFreeAll {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args&, Acc&) {
    dsr_destroy_ro(h, make_handle(T, h.types[T].cap, b, s));   // never reads or writes the object
  }
};
// The same two methods in quad form (k_doall_quad): a lane visits 4 slots,
// reads field 0 of all of them with one 128-bit load, and destroys the chosen
// ones with one block-aggregated mask (lanes of the same block combine into
// one atomicAnd: 1 per 64-slot block instead of 2 for a 32-lane warp).
struct MbFreeOddQ {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void run4(const DevHeap& h, uint32_t T, uint32_t b, uint32_t q, uint32_t m4,
                                              const Args&, Acc&) {
    const uint4 v = __ldcs(quad_u32(h, T, 0, b, q));
    const uint32_t odd = (v.x & 1u) | ((v.y & 1u) << 1) | ((v.z & 1u) << 2) | ((v.w & 1u) << 3);
    dsr_destroy_mask<false>(h, T, b, (uint64_t)(odd & m4) << (4 * q));   // control-dependent on the read
  }
};
struct MbFreeAllQ {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void run4(const DevHeap& h, uint32_t T, uint32_t b, uint32_t q, uint32_t m4,
                                              const Args&, Acc&) {
    dsr_destroy_mask<false>(h, T, b, (uint64_t)m4 << (4 * q));           // never reads or writes the objects
  }
};
// MbFreeAll in block form (k_doall_block): the lane that owns a block
// destroys all its visited objects with one block_free (Alg. 7 + Alg. 2 for
// the whole mask; the objects are never read or written, so no release)
struct MbFreeAllB {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void runb(const DevHeap& h, uint32_t T, uint32_t b, uint64_t m, const Args&, Acc&) {
    block_free<false>(h, T, b, m);
    stat_add(h, ST_FREES, __popcll(m));
  }
};
// MbFreeOdd in block form: the lane reads column 0 of its block's visited
// quads (independent 128-bit loads, all in flight) and frees the odd ones
// with one block_free (control-dependent on the loads: no release)
struct MbFreeOddB {
  struct Args { uint64_t unused; };
  DSR_NO_ACC
  static __device__ __forceinline__ void runb(const DevHeap& h, uint32_t T, uint32_t b, uint64_t m, const Args&, Acc&) {
    const uint4* col = quad_u32(h, T, 0, b, 0);
    uint64_t kill = 0;
#pragma unroll
    for (uint32_t q = 0; q < 16; ++q) {
      if ((m >> (4 * q)) & 0xFull) {
        const uint4 v = __ldg(col + q);
        kill |= (uint64_t)((v.x & 1u) | ((v.y & 1u) << 1) | ((v.z & 1u) << 2) | ((v.w & 1u) << 3)) << (4 * q);
      }
    }
    kill &= m;
    if (kill) {
      block_free<false>(h, T, b, kill);
      stat_add(h, ST_FREES, __popcll(kill));
    }
  }
};
// handle collection (tests): out[atomic++] = this
struct Collect {
  typedef dsr_collect_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const unsigned long long k = atomicAdd((unsigned long long*)a.count, 1ull);
    a.out[k] = make_handle(T, h.types[T].cap, b, s);
  }
};

// ---- Linux Scalability: n allocations per thread, then a free kernel
__global__ void k_ls_alloc(DevHeap h, uint64_t nthreads, dsr_ls_args a) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  for (uint32_t i = 0; i < a.per_thread; ++i) a.handles[t * a.per_thread + i] = dsr_new(h, a.type);
}
__global__ void k_ls_free(DevHeap h, uint64_t nthreads, dsr_ls_args a) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  for (uint32_t i = 0; i < a.per_thread; ++i) dsr_destroy(h, a.handles[t * a.per_thread + i]);
}

// ---- single-thread replay (parity with the oracle's sequential model)
__global__ void k_replay(DevHeap h, dsr_replay_args a) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (uint64_t i = 0; i < a.nops; ++i) {
    const uint32_t op = a.ops[2 * i], arg = a.ops[2 * i + 1];
    if (op == 0) {
      a.handles_out[i] = dsr_new(h, arg);
    } else {
      dsr_destroy(h, a.handles_out[arg]);
      a.handles_out[i] = 0;
    }
  }
}

// ---- concurrent torture: random new/destroy from divergent lanes with
// canaries in the first and last field of every object
__global__ void __launch_bounds__(256) k_torture(DevHeap h, uint64_t nthreads, dsr_torture_args a) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  uint64_t mine[8];
  uint32_t tag[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { mine[k] = 0; tag[k] = 0; }
  uint64_t errs = 0;
  for (uint32_t it = 0; it < a.iters; ++it) {
    const uint64_t r = rng_key(a.seed, t, 9, it);
    const uint32_t k = (uint32_t)(r & 7);
    uint64_t cur = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) if ((uint32_t)j == k) cur = mine[j];
    if (cur) {
      const uint32_t T = h_type(cur);
      const uint32_t last = h.types[T].nfields - 1;
      uint32_t want = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) if ((uint32_t)j == k) want = tag[j];
      if (*field_ptr<uint32_t>(h, cur, 0) != (uint32_t)t || *field_ptr<uint32_t>(h, cur, last) != want) ++errs;
      dsr_destroy(h, cur);
#pragma unroll
      for (int j = 0; j < 8; ++j) if ((uint32_t)j == k) mine[j] = 0;
    } else {
      const uint32_t T = (uint32_t)((r >> 8) % h.ntypes);
      const uint64_t hd = dsr_new(h, T);
      if (hd) {
        const uint32_t w = (uint32_t)(r >> 32) | 1u;
        *field_ptr<uint32_t>(h, hd, 0) = (uint32_t)t;
        *field_ptr<uint32_t>(h, hd, h.types[T].nfields - 1) = w;
#pragma unroll
        for (int j = 0; j < 8; ++j) if ((uint32_t)j == k) { mine[j] = hd; tag[j] = w; }
      }
    }
  }
  for (int j = 0; j < 8; ++j) {
    if (mine[j]) {
      const uint32_t T = h_type(mine[j]);
      if (*field_ptr<uint32_t>(h, mine[j], 0) != (uint32_t)t ||
          *field_ptr<uint32_t>(h, mine[j], h.types[T].nfields - 1) != tag[j]) ++errs;
      if (!a.keep) { dsr_destroy(h, mine[j]); mine[j] = 0; }
    }
    if (a.ledger) a.ledger[t * 8 + j] = mine[j];
  }
  if (errs && a.errors) atomicAdd((unsigned long long*)a.errors, (unsigned long long)errs);
}

// ---- inheritance: a hierarchy rooted at {u32 id, u32 acc}
// a subtype's own field f (f >= 2) holds (id * (f + 1)) truncated to its size
__device__ __forceinline__ uint64_t inh_own(uint32_t id, uint32_t f, uint32_t bytes) {
  const uint64_t v = (uint64_t)id * (f + 1);
  return bytes >= 8 ? v : (v & ((1ull << (8 * bytes)) - 1ull));
}
__device__ __forceinline__ void inh_store(const DevHeap& h, uint64_t hd, uint32_t f, uint64_t v) {
  switch (h.types[h_type(hd)].fsize[f]) {
    case 1: *field_ptr<uint8_t>(h, hd, f) = (uint8_t)v; break;
    case 2: *field_ptr<uint16_t>(h, hd, f) = (uint16_t)v; break;
    case 4: *field_ptr<uint32_t>(h, hd, f) = (uint32_t)v; break;
    default: *field_ptr<uint64_t>(h, hd, f) = v; break;
  }
}
__device__ __forceinline__ uint64_t inh_load(const DevHeap& h, uint32_t T, uint32_t f, uint32_t b, uint32_t s) {
  switch (h.types[T].fsize[f]) {
    case 1: return *field_ptr<uint8_t>(h, T, f, b, s);
    case 2: return *field_ptr<uint16_t>(h, T, f, b, s);
    case 4: return *field_ptr<uint32_t>(h, T, f, b, s);
    default: return *field_ptr<uint64_t>(h, T, f, b, s);
  }
}
__device__ __forceinline__ uint64_t inh_construct(const DevHeap& h, uint32_t T, uint32_t id, bool want) {
  const uint64_t hd = dsr_new_bulk(h, T, want);
  if (hd) {
    *field_ptr<uint32_t>(h, hd, 0) = id;              // inherited columns 0, 1
    *field_ptr<uint32_t>(h, hd, 1) = 0;
    for (uint32_t f = 2; f < h.types[T].nfields; ++f) inh_store(h, hd, f, inh_own(id, f, h.types[T].fsize[f]));
  }
  return hd;
}
__global__ void __launch_bounds__(256) k_inh_new(DevHeap h, uint64_t n, dsr_inh_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    const uint64_t hd = inh_construct(h, (uint32_t)(i % a.ntypes), (uint32_t)i, i < n);
    if (i < n) a.handles[i] = hd;
  }
}
// reads through "base-typed" handles: the column of an inherited field is
// found from the handle's runtime type alone
__global__ void k_inh_read(DevHeap h, uint64_t n, dsr_inh_args a) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t hd = a.handles[i];
    uint64_t v = hd ? *field_ptr<uint32_t>(h, hd, 1) : 0;
    for (uint32_t k = 0; k < h.ntypes; ++k) v |= (uint64_t)dsr_is_a(h, hd, k) << (32 + k);
    a.vals[i] = v;
  }
}
struct InhBump {   // acc = 3 acc + id, inherited fields only
  typedef dsr_inh_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args&, Acc&) {
    uint32_t* acc = field_ptr<uint32_t>(h, T, 1, b, s);
    *acc = 3u * *acc + *field_ptr<uint32_t>(h, T, 0, b, s);
  }
};
struct InhSum {    // per runtime type: count, acc + own fields
  typedef dsr_inh_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    unsigned long long v = *field_ptr<uint32_t>(h, T, 1, b, s);
    for (uint32_t f = 2; f < h.types[T].nfields; ++f) v += inh_load(h, T, f, b, s);
    atomicAdd(a.out + 2 * T, 1ull);
    atomicAdd(a.out + 2 * T + 1, v);
  }
};
struct InhSpawn {  // visits the pre-pass objects only, although it creates objects of the whole subtree
  typedef dsr_inh_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    atomicAdd(a.out, 1ull);
    const uint32_t id = *field_ptr<uint32_t>(h, T, 0, b, s);
    inh_construct(h, (T + 1) % h.ntypes, a.spawn_id0 + id, true);
  }
};

// ------------------------------------------------------------------ tables
bool mb_method_info(uint32_t id, MethodInfo* mi) {
  switch (id) {
    case DSR_M_MB_REDUCE: *mi = {0, sizeof(dsr_mb_reduce_args)}; return true;
    case DSR_M_MB_FREE_ODD: *mi = {DSR_MB_FREEODD_SNAP, 0}; return true;      // self-delete
    case DSR_M_MB_FREE_ALL: *mi = {3, 0}; return true;      // frees whole blocks: blocked distribution
    case DSR_M_COLLECT: *mi = {0, sizeof(dsr_collect_args)}; return true;
    case DSR_M_INH_BUMP: case DSR_M_INH_SUM: *mi = {0, sizeof(dsr_inh_args)}; return true;
    case DSR_M_INH_SPAWN: *mi = {1, sizeof(dsr_inh_args)}; return true;
  }
  return false;
}

bool mb_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  static const uint64_t zero[2] = {0, 0};
  switch (id) {
    case DSR_M_MB_REDUCE: {
      if (c.rk >= 0) return false;                       // single-type passes only
      const dsr_mb_reduce_args* a = (const dsr_mb_reduce_args*)args;
      const uint32_t nf = c.h.types[T].nfields;
      unsigned long long* o = (unsigned long long*)a->out3;
      if (c.h.types[T].cap % 4 != 0) return false;
      for (uint32_t f = 0; f < nf; ++f)
        if (c.h.types[T].fsize[f] != 4) return false;
      switch (nf) {
        case 1: k_mb_reduce<1><<<persistent_grid(c, k_mb_reduce<1>), 256, 0, c.st>>>(c.h, T, o); break;
        case 2: k_mb_reduce<2><<<persistent_grid(c, k_mb_reduce<2>), 256, 0, c.st>>>(c.h, T, o); break;
        case 3: k_mb_reduce<3><<<persistent_grid(c, k_mb_reduce<3>), 256, 0, c.st>>>(c.h, T, o); break;
        case 4: k_mb_reduce<4><<<persistent_grid(c, k_mb_reduce<4>), 256, 0, c.st>>>(c.h, T, o); break;
        case 6: k_mb_reduce<6><<<persistent_grid(c, k_mb_reduce<6>), 256, 0, c.st>>>(c.h, T, o); break;
        case 8: k_mb_reduce<8><<<persistent_grid(c, k_mb_reduce<8>), 256, 0, c.st>>>(c.h, T, o); break;
        case 16: k_mb_reduce<16><<<persistent_grid(c, k_mb_reduce<16>), 256, 0, c.st>>>(c.h, T, o); break;
        default: return false;
      }
      count_launch();
      return true;
    }
    case DSR_M_MB_FREE_ODD:
      if (c.h.flags & DSR_F_SCALAR_DOALL) launch_doall<MbFreeOdd>(c, T, snapshot, zero);
      else if (c.h.flags & DSR_F_QUAD_FREE) launch_doall_quad<MbFreeOddQ>(c, T, snapshot, zero);
      else launch_doall_block<MbFreeOddB>(c, T, snapshot, zero);
      return true;
    case DSR_M_MB_FREE_ALL:
      if (c.h.flags & DSR_F_SCALAR_DOALL) launch_doall<MbFreeAll>(c, T, snapshot, zero);
      else if (c.h.flags & DSR_F_QUAD_FREE) launch_doall_quad<MbFreeAllQ>(c, T, snapshot, zero);
      else launch_doall_block<MbFreeAllB>(c, T, snapshot, zero);
      return true;
    case DSR_M_COLLECT: launch_doall<Collect>(c, T, snapshot, args); return true;
    case DSR_M_INH_BUMP: case DSR_M_INH_SUM: case DSR_M_INH_SPAWN:
      for (uint32_t t = 0; t < c.h.ntypes; ++t)       // every type derives from a root {u32 id, u32 acc}
        if (c.h.types[t].nfields < 2 || c.h.types[t].fsize[0] != 4 || c.h.types[t].fsize[1] != 4) return false;
      if (id == DSR_M_INH_BUMP) launch_doall<InhBump>(c, T, snapshot, args);
      else if (id == DSR_M_INH_SUM) launch_doall<InhSum>(c, T, snapshot, args);
      else launch_doall<InhSpawn>(c, T, snapshot, args);
      return true;
  }
  return false;
}

bool mb_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  switch (id) {
    case DSR_K_MB_NEW: {
      if (bytes != sizeof(dsr_mb_new_args) || c.h.ntypes < 3) { *ok = 0; return true; }
      {
        const dsr_mb_new_args& ma = *(const dsr_mb_new_args*)args;
        // (__launch_bounds__ minimum 8 / 6 / 4 CTAs per SM measured equal: 9.2-9.6 ms)
        if (ma.in && ((ma.t0 & 3) || ma.in_host)) { *ok = 0; return true; }   // host inputs are staged by dsr_launch
        if (c.h.flags & DSR_F_CTA_NEW) {
          if (ma.in) { *ok = 0; return true; }
          k_mb_new<true, 8><<<grid_for(c, n, k_mb_new<true, 8>), 256, 0, c.st>>>(c.h, n, ma);
        } else {
          if (cudaMemsetAsync(&c.h.ctrl[CTRL_WORK], 0, 8, c.st) != cudaSuccess) { *ok = 0; return true; }
          if (ma.in) k_mb_new<false, DSR_MB_MINB, true><<<grid_for(c, n, k_mb_new<false, DSR_MB_MINB, true>), 256, 0, c.st>>>(c.h, n, ma);
          else k_mb_new<false, DSR_MB_MINB><<<grid_for(c, n, k_mb_new<false, DSR_MB_MINB>), 256, 0, c.st>>>(c.h, n, ma);
        }
      }
      count_launch();
      return true;
    }
    case DSR_K_MB_NEW_BULK: {
      if (bytes != sizeof(dsr_mb_new_args) || c.h.ntypes < 3) { *ok = 0; return true; }
      const dsr_mb_new_args& ma = *(const dsr_mb_new_args*)args;
      if (ma.in && ((ma.t0 & 3) || ma.in_host)) { *ok = 0; return true; }   // host inputs are staged by dsr_launch
      for (uint32_t t = 0; t < 3; ++t)                  // A{3 x u32}, B{4 x u32}, C{6 x u32}
        if (c.h.types[t].nfields != 3u + t + (t == 2) || c.h.types[t].fsize[0] != 4) { *ok = 0; return true; }
      if (cudaMemsetAsync(&c.h.ctrl[CTRL_WORK], 0, 8, c.st) != cudaSuccess) { *ok = 0; return true; }
      if (ma.in) k_mb_new_bulk<true><<<grid_for(c, n, k_mb_new_bulk<true>), 256, 0, c.st>>>(c.h, n, ma);
      else k_mb_new_bulk<false><<<grid_for(c, n, k_mb_new_bulk<false>), 256, 0, c.st>>>(c.h, n, ma);
      count_launch();
      return true;
    }
    case DSR_K_LS_ALLOC:
    case DSR_K_LS_FREE: {
      if (bytes != sizeof(dsr_ls_args)) { *ok = 0; return true; }
      const dsr_ls_args a = *(const dsr_ls_args*)args;
      if (a.type >= c.h.ntypes) { *ok = 0; return true; }
      const int g = (int)((n + 255) / 256);
      if (id == DSR_K_LS_ALLOC) k_ls_alloc<<<g, 256, 0, c.st>>>(c.h, n, a);
      else k_ls_free<<<g, 256, 0, c.st>>>(c.h, n, a);
      count_launch();
      return true;
    }
    case DSR_K_INH_NEW:
    case DSR_K_INH_READ: {
      if (bytes != sizeof(dsr_inh_args)) { *ok = 0; return true; }
      const dsr_inh_args a = *(const dsr_inh_args*)args;
      for (uint32_t t = 0; t < c.h.ntypes; ++t)       // every type derives from a root {u32 id, u32 acc}
        if (c.h.types[t].nfields < 2 || c.h.types[t].fsize[0] != 4 || c.h.types[t].fsize[1] != 4) { *ok = 0; return true; }
      if (id == DSR_K_INH_NEW) {
        if (a.ntypes < 1 || a.ntypes > c.h.ntypes || !a.handles) { *ok = 0; return true; }
        k_inh_new<<<grid_for(c, n, k_inh_new), 256, 0, c.st>>>(c.h, n, a);
      } else {
        if (!a.handles || !a.vals) { *ok = 0; return true; }
        k_inh_read<<<grid_for(c, n, k_inh_read), 256, 0, c.st>>>(c.h, n, a);
      }
      count_launch();
      return true;
    }
    case DSR_K_REPLAY: {
      if (bytes != sizeof(dsr_replay_args)) { *ok = 0; return true; }
      k_replay<<<1, 1, 0, c.st>>>(c.h, *(const dsr_replay_args*)args);
      count_launch();
      return true;
    }
    case DSR_K_TORTURE: {
      if (bytes != sizeof(dsr_torture_args)) { *ok = 0; return true; }
      for (uint32_t t = 0; t < c.h.ntypes; ++t)
        for (uint32_t f = 0; f < c.h.types[t].nfields; ++f)
          if (f == 0 || f == c.h.types[t].nfields - 1)
            if (c.h.types[t].fsize[f] != 4) { *ok = 0; return true; }
      k_torture<<<(int)((n + 255) / 256), 256, 0, c.st>>>(c.h, n, *(const dsr_torture_args*)args);
      count_launch();
      return true;
    }
  }
  return false;
}

}  // namespace dsr
