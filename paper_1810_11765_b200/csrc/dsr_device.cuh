// dsr_device.cuh -- device side of the B200 DynaSOAr hot path (sm_100a).
//
// Lock-free hierarchical bitmaps, block heap with slot
// reservation / freeing / invalidation (App. A) and the
// warp-aggregated object allocator (Algs. 1-2 P:375-426, request coalescing
// and bitmap rotation P:646-654, n-th set bit P:689).
//
// Memory model (reading R-MEMORY / C21): bitmap words are modified with 64-bit
// device-scope atomics; plain reads of shared words are ld.relaxed.gpu.
// initialize_block stores the type id, then the object bitmap with
// st.release (the paper's "volatile write; threadfence; volatile write",
// Alg. 8); slot reservation and invalidation use atom.acquire so the type id
// and the fields read afterwards are those of the initialised block (Alg. 1
// l.10, footnote P:1091); a slot free uses atom.release so the freeing lanes'
// last reads/writes of the objects precede any reuse of the slots.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/dsr.h"

namespace dsr {

typedef unsigned long long ull;

struct DevBitmap {
  uint64_t* lvl[DSR_MAX_LEVELS];   // level 0 = leaf containers
  uint32_t nlevels;
  uint32_t pad_;
  uint64_t nbits;
  unsigned long long* err;         // the heap's sticky error word (debug builds: bounded spins)
};

struct DevType {
  uint32_t cap;                    // N_T
  uint32_t nfields;
  uint32_t parent;                 // 0 = none, k = derives from type k - 1
  uint32_t pad_;
  uint64_t valid;                  // low N_T bits
  uint64_t pad;                    // ~valid: padding bits kept at 1
  uint32_t fsize[DSR_MAX_FIELDS];
  uint32_t col_off[DSR_MAX_FIELDS];
};

// control page word offsets (u64 units) -- DESIGN.md "HBM layout"
// CTRL_RBEG + k: begin of the k-th type's range of R in a subtree do-all (k <= DSR_MAX_TYPES)
// CTRL_WORK: dynamic work counter of persistent user kernels
enum { CTRL_ERR = 0, CTRL_RCOUNT = 1, CTRL_SCRATCH = 2, CTRL_WORK = 3, CTRL_RBEG = 4, CTRL_STATS = 16, CTRL_AUDIT = 40 };
// ERRB_BOUNDS: a debug build's bounds check failed (an object access outside
// the heap's blocks / a type's slots or fields, dsr_poll_error -> DSR_ERR_INVARIANT)
enum { ERRB_OOM = 1, ERRB_BUDGET = 2, ERRB_BOUNDS = 4 };
// control-page words 480..511: where a debug build redirects an out-of-bounds access
enum { CTRL_SINK = 480 };
enum { ST_ALLOCS = 0, ST_FREES, ST_INITS, ST_BFREES, ST_ROLLBACKS, ST_INVFAIL, ST_RESRETRY, ST_OOM,
       ST_REQ, ST_FIND, ST_FINDFAIL, ST_RESZERO, ST_CYC_FIND, ST_CYC_SLOW, ST_CYC_RES, ST_CYC_REQ, ST_HINTZERO,
       ST_N };

struct DevHeap {
  uint8_t* data;          // M * block_bytes SOA data segments
  uint64_t* alloc_bm;     // object allocation bitmap per block
  uint64_t* iter_bm;      // object iteration bitmap per block
  uint8_t* type;          // type id per block, 1-based, 0 = never initialised
  uint32_t* R;            // do-all block list
  ull* ctrl;              // control page
  uint32_t* hints;        // per hardware warp slot and type: the block it last allocated from
  uint32_t M;
  uint32_t block_bytes;
  uint32_t ntypes;
  uint32_t r_attempts;
  uint32_t flags;
  uint32_t hint_mask;     // hint slots - 1 (power of two)
  uint32_t sms;           // SM count (SM-affine rotation)
  uint32_t pad2_;
  uint64_t seed;
  DevBitmap freebm;
  DevBitmap allocbm[DSR_MAX_TYPES];
  DevBitmap activebm[DSR_MAX_TYPES];
  DevType types[DSR_MAX_TYPES];
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.relaxed.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u8 [%0], %1;" ::"l"(p), "h"((uint16_t)v) : "memory");
}
__device__ __forceinline__ uint64_t atom_or(uint64_t* p, uint64_t m) { return atomicOr((ull*)p, (ull)m); }
__device__ __forceinline__ uint64_t atom_and(uint64_t* p, uint64_t m) { return atomicAnd((ull*)p, (ull)m); }
// acquire: later reads of the block (type id, fields) are ordered after the RMW
__device__ __forceinline__ uint64_t atom_or_acquire(uint64_t* p, uint64_t m) {
  uint64_t old;
  asm volatile("atom.acquire.gpu.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(m) : "memory");
  return old;
}
// relaxed RMW that is also a compiler barrier (dsr_destroy_ro)
__device__ __forceinline__ uint64_t atom_and_relaxed(uint64_t* p, uint64_t m) {
  uint64_t old;
  asm volatile("atom.relaxed.gpu.global.and.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(m) : "memory");
  return old;
}
// release: earlier reads / writes of the freed objects are ordered before the RMW
__device__ __forceinline__ uint64_t atom_and_release(uint64_t* p, uint64_t m) {
  uint64_t old;
  asm volatile("atom.release.gpu.global.and.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(m) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t rotr64(uint64_t x, uint32_t r) { return r ? (x >> r) | (x << (64 - r)) : x; }
__device__ __forceinline__ uint64_t rotl64(uint64_t x, uint32_t r) { return r ? (x << r) | (x >> (64 - r)) : x; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint64_t shfl64(uint32_t mask, uint64_t v, uint32_t src) {
  uint32_t lo = __shfl_sync(mask, (uint32_t)v, src), hi = __shfl_sync(mask, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
// index of the lowest set bit of x != 0 on 32-bit halves (BREV + FLO on one
// half: 5 fewer instructions than __ffsll's 64-bit negate-and-mask form)
__device__ __forceinline__ uint32_t ctz64(uint64_t x) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return lo ? (uint32_t)__ffs(lo) - 1u : 31u + (uint32_t)__ffs(hi);
}
// 0-based n-th set bit of x, n < popc(x) (P:689 clears the lowest bit n times,
// then ffs).  A single run of ones (a fresh block, a coalesced chunk) is
// answered directly; otherwise a 6-step popc binary search.
__device__ __forceinline__ uint32_t nth_bit(uint64_t x, uint32_t n) {
  const uint32_t lo = ctz64(x);
  const uint64_t run = x >> lo;
  if ((run & (run + 1ull)) == 0) return lo + n;
  uint32_t pos = 0, c = __popc((uint32_t)x);
  if (n >= c) { n -= c; x >>= 32; pos = 32; }
  uint32_t w = (uint32_t)x;
  c = __popc(w & 0xFFFFu); if (n >= c) { n -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xFFu);   if (n >= c) { n -= c; w >>= 8;  pos += 8; }
  c = __popc(w & 0xFu);    if (n >= c) { n -= c; w >>= 4;  pos += 4; }
  c = __popc(w & 0x3u);    if (n >= c) { n -= c; w >>= 2;  pos += 2; }
  return pos + ((n >= (w & 1u)) ? 1u : 0u);
}
__device__ __forceinline__ void backoff(uint32_t& ns) {
  __nanosleep(ns);
  ns = ns < 256 ? ns * 2 : 256;
}
// Debug builds (-DDSR_DEBUG, build(variant="debug")): illegal use (a
// second net set / clear of a bitmap bit; destroying a slot that is
// not allocated) deadlocks in the paper; here a spin gives up after 2^20
// backoffs and the precondition of Alg. 7 is checked, both reported as
// DSR_ERR_RETRY_BUDGET through the sticky error word.
#ifdef DSR_DEBUG
#define DSR_SPIN_GUARD(errp, n)                                         \
  if (++(n) > (1u << 20)) {                                             \
    atomicOr((errp), 2ull /* ERRB_BUDGET */);                           \
    break;                                                              \
  }
#else
#define DSR_SPIN_GUARD(errp, n)
#endif
// Fault-injection builds (-DDSR_FAULT): a pseudo-random pause of 0.5-8 us (up to ~40 us
// after a block was found) at
// the linearisation points between which other threads can interleave
// (found block -> reservation, Alg. 1 l.9; EMPTY -> invalidate, Alg. 2 l.7;
// invalidate -> rollback, Alg. 9 l.8), so that the rare branches -- type
// change rollback (Alg. 1 l.14), failed invalidation and its deferred
// deactivation (Alg. 9 l.8-13) -- run in tests on tiny heaps.
#ifdef DSR_FAULT
__device__ __forceinline__ void fault_point(uint64_t salt) {
  uint64_t z = ((uint64_t)clock64() ^ (salt << 32) ^ (threadIdx.x * 0x9E3779B97F4A7C15ull)) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 31;
  if ((z & 3) == 0) __nanosleep(500 + (uint32_t)((z >> 8) & 7679));
  // a found block held across a long pause: time for it to be emptied, freed
  // and re-initialised for another type (the type-change rollback's window)
  if (salt == 1 && (z & 0x70) == 0) for (int k = 0; k < 8; ++k) __nanosleep(4000);
}
#define DSR_FAULT_POINT(salt) fault_point(salt)
#else
#define DSR_FAULT_POINT(salt)
#endif
__device__ __forceinline__ void flag_error(const DevHeap& h, uint32_t bit) { atomicOr(&h.ctrl[CTRL_ERR], (ull)bit); }
__device__ __forceinline__ void stat_add(const DevHeap& h, int which, uint64_t v) {
  if (h.flags & DSR_F_STATS) atomicAdd(&h.ctrl[CTRL_STATS + which], (ull)v);
}

// counter-based RNG, reading R-RNG (SplitMix64 output function)
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t step, uint64_t phase, uint64_t idx) {
  return sm64(sm64(sm64(seed) ^ step) ^ ((phase << 40) | idx));
}
// the same key with the (seed, step) prefix sm64(sm64(seed) ^ step) hoisted out of a loop
__device__ __forceinline__ uint64_t rng_prefix(uint64_t seed, uint64_t step) { return sm64(sm64(seed) ^ step); }
__device__ __forceinline__ uint64_t rng_key_p(uint64_t prefix, uint64_t phase, uint64_t idx) {
  return sm64(prefix ^ ((phase << 40) | idx));
}

// ------------------------------------------------------------------ handles (Fig. 5, Listing 2)
__device__ __forceinline__ uint64_t make_handle(uint32_t T, uint32_t cap, uint32_t bid, uint32_t slot) {
  return ((uint64_t)(T + 1) << 56) | ((uint64_t)(cap - 1) << 50) | ((uint64_t)bid << 6) | slot;
}
__device__ __forceinline__ uint32_t h_slot(uint64_t h) { return (uint32_t)(h & 0x3Full); }
__device__ __forceinline__ uint32_t h_bid(uint64_t h) { return (uint32_t)((h & 0x3FFFFFFFFFFC0ull) >> 6); }
__device__ __forceinline__ uint32_t h_type(uint64_t h) { return (uint32_t)(h >> 56) - 1u; }  // 0-based
__device__ __forceinline__ bool h_is(uint64_t h, uint32_t T) { return (h >> 56) == (uint64_t)(T + 1); }

// Debug builds (-DDSR_DEBUG): every object access through field_ptr is
// bounds-checked -- type, field, block index and slot -- and an access that
// fails is reported (ERRB_BOUNDS) and redirected to a sink in the control
// page instead of touching memory outside the heap's blocks (the own-checks
// replacement for compute-sanitizer memcheck, which this pool does not run).
#ifdef DSR_DEBUG
__device__ __forceinline__ bool dbg_obj_ok(const DevHeap& h, uint32_t T, uint32_t f, uint32_t bid, uint32_t slot) {
  return T < h.ntypes && f < h.types[T].nfields && bid < h.M && slot < h.types[T].cap;
}
#endif
template <class V>
__device__ __forceinline__ V* field_ptr(const DevHeap& h, uint32_t T, uint32_t f, uint32_t bid, uint32_t slot) {
#ifdef DSR_DEBUG
  if (!dbg_obj_ok(h, T, f, bid, slot)) {
    atomicOr(&h.ctrl[CTRL_ERR], (unsigned long long)ERRB_BOUNDS);
    return reinterpret_cast<V*>(&h.ctrl[CTRL_SINK]);
  }
#endif
  // Listing 2: block + field_offset * capacity + slot * sizeof
  return reinterpret_cast<V*>(h.data + (size_t)bid * h.block_bytes + h.types[T].col_off[f]) + slot;
}
template <class V>
__device__ __forceinline__ V* field_ptr(const DevHeap& h, uint64_t hd, uint32_t f) {
  return field_ptr<V>(h, h_type(hd), f, h_bid(hd), h_slot(hd));
}

// instance-of: the runtime type from the handle bits, then up the
// parent chain (inheritance).  A base field is the same column index
// in every subtype, so field_ptr(h, handle, f) reads it through any handle.
__device__ __forceinline__ bool dsr_is_a(const DevHeap& h, uint64_t hd, uint32_t T) {
  if (hd == 0) return false;
  uint32_t t = h_type(hd);
#pragma unroll 1
  for (int k = 0; k < DSR_MAX_TYPES; ++k) {
    if (t == T) return true;
    const uint32_t p = h.types[t].parent;
    if (!p) return false;
    t = p - 1;
  }
  return false;
}

// ------------------------------------------------------------------ rotation (reading R-ROT / C3)
__device__ __forceinline__ uint64_t rot_hash(const DevHeap& h, uint64_t who, uint64_t retry) {
  if (h.flags & DSR_F_NO_ROTATE) return 0;
  // one multiply-xorshift round (any function is a correct rotation, C3; the
  // full SplitMix64 finaliser cost ~6 % of new1 once the allocation kernel
  // became issue-bound: 6.1 -> 5.75 ms)
  const uint64_t z = (who ^ (retry << 40) ^ h.seed) * 0x9E3779B97F4A7C15ull;
  return z ^ (z >> 29);
}
__device__ __forceinline__ uint64_t warp_gid() {
  return ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}
// hint table slot of the calling hardware warp (SM id x warp slot; a stale or
// shared slot only degrades the hint, never correctness)
__device__ __forceinline__ volatile uint32_t* hint_slot(const DevHeap& h, uint32_t T) {
  uint32_t smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  return h.hints + (((smid << 6) | (wid & 63)) & h.hint_mask) * DSR_MAX_TYPES + T;
}

// first set bit of c at or after position r, cyclically (c != 0): the same
// result as ffs(rotr(c, r)) + r mod 64 (the rotated search) without the
// 64-bit rotate
__device__ __forceinline__ uint32_t ffs_from(uint64_t c, uint32_t r) {
  const uint64_t hi = c & (~0ull << r);
  return ctz64(hi ? hi : c);
}

// ------------------------------------------------------------------ hierarchical bitmap
// set(pos) at level l: "switches the bit from 0 to 1, retries until the bit
// was changed"; cascades set-first upward (Def. P:1129).  Upper
// levels always use the retrying versions.
__device__ __forceinline__ void bm_set_from(const DevBitmap& b, uint32_t l, uint64_t pos) {
  for (; l < b.nlevels; ++l) {
    uint64_t* w = b.lvl[l] + (pos >> 6);
    const uint64_t m = 1ull << (pos & 63);
    uint64_t prev = atom_or(w, m);     // first try blind (legal use: the bit is 0)
    uint32_t ns = 32, spins = 0;
    while (prev & m) {
      DSR_SPIN_GUARD(b.err, spins)
      backoff(ns);   // an in-flight clear of this bit is pending: wait for it, then retry
      if (!(ld_relaxed(w) & m)) prev = atom_or(w, m);
    }
    if (prev != 0) return;     // not set-first: upper level already 1
    pos >>= 6;
  }
}
__device__ __forceinline__ void bm_clear_from(const DevBitmap& b, uint32_t l, uint64_t pos) {
  for (; l < b.nlevels; ++l) {
    uint64_t* w = b.lvl[l] + (pos >> 6);
    const uint64_t m = 1ull << (pos & 63);
    uint64_t prev = atom_and(w, ~m);   // first try blind (legal use: the bit is 1)
    uint32_t ns = 32, spins = 0;
    while (!(prev & m)) {
      DSR_SPIN_GUARD(b.err, spins)
      backoff(ns);   // an in-flight set of this bit is pending
      if (ld_relaxed(w) & m) prev = atom_and(w, ~m);
    }
    if (prev != m) return;     // Alg. 3 l.6: cascade only if popc(prev) = 1
    pos >>= 6;
  }
}
// the rest of a level-0 bm_clear / bm_set whose blind first atomic returned `prev`
__device__ __forceinline__ void bm_clear_finish(const DevBitmap& b, uint64_t pos, uint64_t prev) {
  uint64_t* w = b.lvl[0] + (pos >> 6);
  const uint64_t m = 1ull << (pos & 63);
  uint32_t ns = 32, spins = 0;
  while (!(prev & m)) {
    DSR_SPIN_GUARD(b.err, spins)
    backoff(ns);
    if (ld_relaxed(w) & m) prev = atom_and(w, ~m);
  }
  if (prev == m && b.nlevels > 1) bm_clear_from(b, 1, pos >> 6);
}
__device__ __forceinline__ void bm_set_finish(const DevBitmap& b, uint64_t pos, uint64_t prev) {
  uint64_t* w = b.lvl[0] + (pos >> 6);
  const uint64_t m = 1ull << (pos & 63);
  uint32_t ns = 32, spins = 0;
  while (prev & m) {
    DSR_SPIN_GUARD(b.err, spins)
    backoff(ns);
    if (!(ld_relaxed(w) & m)) prev = atom_or(w, m);
  }
  if (prev == 0 && b.nlevels > 1) bm_set_from(b, 1, pos >> 6);
}
__device__ __forceinline__ void bm_set(const DevBitmap& b, uint64_t pos) { bm_set_from(b, 0, pos); }
__device__ __forceinline__ void bm_clear(const DevBitmap& b, uint64_t pos) { bm_clear_from(b, 0, pos); }

// Alg. 3 (try_clear) and its symmetric try_set
__device__ __forceinline__ bool bm_try_clear(const DevBitmap& b, uint64_t pos) {
  uint64_t* w = b.lvl[0] + (pos >> 6);
  const uint64_t m = 1ull << (pos & 63);
  const uint64_t prev = atom_and(w, ~m);
  if (!(prev & m)) return false;
  if (prev == m && b.nlevels > 1) bm_clear_from(b, 1, pos >> 6);
  return true;
}
__device__ __forceinline__ bool bm_try_set(const DevBitmap& b, uint64_t pos) {
  uint64_t* w = b.lvl[0] + (pos >> 6);
  const uint64_t m = 1ull << (pos & 63);
  const uint64_t prev = atom_or(w, m);
  if (prev & m) return false;
  if (prev == 0 && b.nlevels > 1) bm_set_from(b, 1, pos >> 6);
  return true;
}
__device__ __forceinline__ bool bm_get(const DevBitmap& b, uint64_t pos) {
  return (ld_relaxed(b.lvl[0] + (pos >> 6)) >> (pos & 63)) & 1;
}

// Alg. 4 try_find_set, top-down; each level's container is rotated by 6
// bits of `rh` before ffs.  May FAIL spuriously.
__device__ __forceinline__ int64_t bm_try_find_set(const DevBitmap& b, uint64_t rh, uint64_t* leaf = nullptr) {
  uint64_t cid = 0;
  for (int l = (int)b.nlevels - 1; l >= 0; --l) {
    const uint64_t c = ld_relaxed(b.lvl[l] + cid);
    if (c == 0) return -1;
    const uint32_t r = (uint32_t)(rh >> (6 * l)) & 63u;
    const uint32_t i = ffs_from(c, r);
    cid = cid * 64 + i;
    if (l == 0 && leaf) *leaf = c;     // the leaf container the result came from
  }
  return (int64_t)cid;
}
// SM-affine rotation ("rotating-shifted by a value depending on the warp
// ID and a seed"): the warps of SM s start every search inside their own
// contiguous range of level-1 containers, so concurrent searches and new
// blocks of different SMs land in different containers and cache lines.
__device__ __forceinline__ void home_range(const DevBitmap& b, uint32_t sms, uint32_t* lo, uint32_t* len) {
  const uint32_t n1 = (uint32_t)(((((uint64_t)b.nbits + 63) >> 6) + 63) >> 6);
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid %= sms;
  uint32_t a = (uint32_t)((uint64_t)smid * n1 / sms), e = (uint32_t)((uint64_t)(smid + 1) * n1 / sms);
  if (e <= a) { a = a < n1 ? a : n1 - 1; e = a + 1; }      // small heaps: SMs share containers
  *lo = a;
  *len = e - a;
}
// try_find_set restricted to the home range (levels 1 and 0, rotated); -1 if
// the probed containers are empty (the caller then counts a failed attempt)
__device__ __forceinline__ int64_t bm_find_home(const DevBitmap& b, uint32_t lo, uint32_t len, uint64_t rh,
                                                uint64_t* leaf = nullptr) {
  const uint32_t start = (uint32_t)(rh % len);
  for (uint32_t k = 0; k < len && k < 8; ++k) {
    const uint32_t i1 = lo + (start + k) % len;
    const uint64_t c1 = ld_relaxed(b.lvl[1] + i1);
    if (!c1) continue;
    const uint32_t r1 = (uint32_t)(rh >> 8) & 63u;
    const uint64_t i0 = (uint64_t)i1 * 64 + ((((uint32_t)__ffsll((long long)rotr64(c1, r1))) - 1u + r1) & 63u);
    const uint64_t c0 = ld_relaxed(b.lvl[0] + i0);
    if (!c0) continue;
    const uint32_t r0 = (uint32_t)(rh >> 14) & 63u;
    if (leaf) *leaf = c0;
    return (int64_t)(i0 * 64 + ((((uint32_t)__ffsll((long long)rotr64(c0, r0))) - 1u + r0) & 63u));
  }
  return -1;
}
// next set bit of the leaf container `c` after position pos (cyclic), -1 if none
__device__ __forceinline__ int64_t leaf_next(uint64_t c, uint64_t pos) {
  const uint32_t p = (uint32_t)(pos & 63);
  c &= ~(1ull << p);
  if (c == 0) return -1;
  const uint32_t r = (p + 1) & 63u;
  const uint32_t i = ffs_from(c, r);
  return (int64_t)((pos & ~63ull) | i);
}
// clear(): find + try_clear until the clear succeeds (reading R-CLEARANY).
// Used on the free bitmap only.  The rotation there applies to the lowest
// DSR_FREE_ROT_LEVELS levels (reading R-FREEROT); above them the search takes
// the lowest container with a free block, so new blocks fill the heap from its
// low end instead of being scattered over all of it: the blocks an app uses
// then span a range set by the live data, not by the heap size.
#ifndef DSR_FREE_ROT_LEVELS
#define DSR_FREE_ROT_LEVELS 3
#endif
constexpr uint64_t kFreeRotMask = DSR_FREE_ROT_LEVELS >= 10 ? ~0ull : ((1ull << (6 * DSR_FREE_ROT_LEVELS)) - 1ull);
__device__ __forceinline__ int64_t bm_clear_any(const DevHeap& h, const DevBitmap& b, uint64_t who, uint64_t retry0) {
  for (uint64_t k = 0;; ++k) {
    const int64_t i = bm_try_find_set(b, rot_hash(h, who, retry0 + k) & kFreeRotMask);
    if (i < 0) return -1;
    if (bm_try_clear(b, (uint64_t)i)) return i;
  }
}

// ------------------------------------------------------------------ blocks (App. A)
// Alg. 8: type <- T; fence; bitmap <- padding mask
__device__ __forceinline__ void init_block(const DevHeap& h, uint32_t T, uint32_t bid) {
  st_relaxed_u8(h.type + bid, T + 1);
  st_release(h.alloc_bm + bid, h.types[T].pad);          // type store ordered before the bitmap store
}

// Alg. 6 generalised to a coalesced multi-slot reservation: pick up to `need`
// free slots (rotated) and set them with ONE atomicOr; returns the
// slots this call actually flipped (may be fewer; 0 = block full/invalidated).
__device__ __forceinline__ uint64_t block_reserve(const DevHeap& h, uint32_t bid, uint32_t need, uint32_t rot,
                                                  uint64_t* before_out, bool known = false, uint64_t known_word = 0) {
  uint64_t* w = h.alloc_bm + bid;
  uint64_t cur = known ? known_word : ld_relaxed(w);  // a block we just initialised: its word is known
  for (;;) {
    const uint64_t fr = ~cur;
    if (fr == 0) return 0;
    uint64_t rf = rotr64(fr, rot);
    if ((uint32_t)__popcll(rf) > need) rf &= (2ull << nth_bit(rf, need - 1)) - 1ull;   // first `need` bits
    const uint64_t sel = rotl64(rf, rot);
    const uint64_t before = atom_or_acquire(w, sel);       // acquire: type id / fields read after
    const uint64_t got = sel & ~before;
    if (got) { *before_out = before; return got; }
    stat_add(h, ST_RESRETRY, 1);
    cur = before | sel;
  }
}

// Alg. 9 (iterative, footnote P:1077) with padding: succeeds iff every
// non-padding bit was 0, i.e. before == pad(t).
// *t_out: the block's type, read while we hold its invalidated bits.
__device__ __forceinline__ bool block_invalidate(const DevHeap& h, uint32_t bid, uint32_t* t_out) {
  uint64_t* w = h.alloc_bm + bid;
  for (;;) {
    const uint64_t before = atom_or_acquire(w, ~0ull);
    if (before == ~0ull) return false;
    const uint32_t t = ld_relaxed_u8(h.type + bid) - 1u;   // fixed while we hold invalidated bits
    const uint64_t pad = h.types[t].pad;
    if (before == pad) { *t_out = t; return true; }
    stat_add(h, ST_INVFAIL, 1);
    DSR_FAULT_POINT(3);
    const uint64_t before_rb = atom_and(w, before);         // rollback exactly our bits
    if (before_rb != ~0ull) bm_clear(h.activebm[t], bid);   // deferred deactivation
    if ((before_rb & before) != pad) return false;          // not empty again
  }
}

// Alg. 7 + Alg. 2 for a mask of slots of one block of type T (coalesced free).
// FIRST iff before == ~0; EMPTY iff the remaining bits are padding only;
// both at once: activate, then invalidate (reading R-FIRSTEMPTY / C17).
// RELEASE = false: the relaxed form for dsr_destroy_ro (no fence).
// USER = false: the rollback of a reservation (Alg. 1 l.14), whose block may
// still be finishing its own allocated.set (debug checks off).
template <bool RELEASE = true, bool USER = true>
__device__ __forceinline__ void block_free(const DevHeap& h, uint32_t T, uint32_t bid, uint64_t mask) {
#ifdef DSR_DEBUG
  // An object's block is in allocated[T] from before the object is handed out
  // until the block is freed, which needs every object destroyed: a destroy
  // into a block that is not allocated is a double destroy whose block was
  // freed (and invalidated to all ones, so the bitmap check below cannot see it).
  if (USER && !bm_get(h.allocbm[T], bid)) {
    atomicOr(&h.ctrl[CTRL_ERR], (ull)ERRB_BUDGET);
    return;
  }
#endif
  uint64_t before = RELEASE ? atom_and_release(h.alloc_bm + bid, ~mask) : atom_and_relaxed(h.alloc_bm + bid, ~mask);
#ifdef DSR_DEBUG
  if (USER && (before & mask) != mask) {    // Alg. 7 precondition: slots not allocated
    atomicOr(&h.ctrl[CTRL_ERR], (ull)ERRB_BUDGET);
    mask &= before;
    if (!mask) return;
  }
#endif
  const bool first = before == ~0ull;
  const bool empty = (before & ~mask) == h.types[T].pad;
  if (first) bm_set(h.activebm[T], bid);
  uint32_t t;
  if (empty) DSR_FAULT_POINT(2);
  if (empty && block_invalidate(h, bid, &t)) {
    // Alg. 2 l.7-11: active[t].clear, allocated[t].clear, free.set -- three
    // independent leaf words, so the three blind first atomics are in flight
    // together; each then finishes (wrong-state retry, upward cascade) as in
    // bm_clear / bm_set.  (One L2 round trip instead of three, plus the type
    // read that block_invalidate already did.)
    const uint64_t m = 1ull << (bid & 63);
    const uint64_t pa = atom_and(h.activebm[t].lvl[0] + (bid >> 6), ~m);
    const uint64_t pl = atom_and(h.allocbm[t].lvl[0] + (bid >> 6), ~m);
    const uint64_t pf = atom_or(h.freebm.lvl[0] + (bid >> 6), m);
    bm_clear_finish(h.activebm[t], bid, pa);
    bm_clear_finish(h.allocbm[t], bid, pl);
    bm_set_finish(h.freebm, bid, pf);
    stat_add(h, ST_BFREES, 1);
  }
}

// A random active block of T near `last` (same leaf word, else a random
// non-empty leaf under the same level-1 word); 0xFFFFFFFF if none.  One or two
// relaxed loads of active[T] instead of a top-down search.
__device__ __forceinline__ uint32_t near_block(const DevHeap& h, uint32_t T, uint32_t last, uint64_t rr) {
  if (last >= h.M) return 0xFFFFFFFFu;
  const uint64_t lw = ld_relaxed(h.activebm[T].lvl[0] + (last >> 6)) & ~(1ull << (last & 63));
  if (lw) return (last & ~63u) | nth_bit(lw, ((((uint32_t)(rr >> 40)) & 63u) * (uint32_t)__popcll(lw)) >> 6);
  if (h.activebm[T].nlevels < 2) return 0xFFFFFFFFu;
  const uint64_t l1 = ld_relaxed(h.activebm[T].lvl[1] + (last >> 12));
  if (!l1) return 0xFFFFFFFFu;
  const uint32_t li = ((last >> 12) << 6) | nth_bit(l1, ((((uint32_t)(rr >> 46)) & 63u) * (uint32_t)__popcll(l1)) >> 6);
  const uint64_t w = ld_relaxed(h.activebm[T].lvl[0] + li);
  return w ? (li << 6) | nth_bit(w, ((((uint32_t)(rr >> 52)) & 63u) * (uint32_t)__popcll(w)) >> 6) : 0xFFFFFFFFu;
}

// Alg. 1 for one coalesced request of `need` slots (leader lane only).
// Returns the reserved slot mask (0 = OOM) and the block in *bid_out.
// An "active block lookup attempt" (Fig. 11) fails when
// try_find_set FAILs or when the block it returned yields no slot (full or
// invalidated meanwhile); after r failed attempts the leader takes the slow
// path (reading R-RETRY).  Sequentially this is exactly Alg. 1.
// The request-level profile (lookups, zero-slot reservations, cycle stamps)
// exists only in a -DDSR_PROFILE build (scripts/gpu_stats.sh): its live
// registers cost the default path spills and ~4 % of its instructions.
static __device__ __forceinline__ uint64_t reserve_chunk(const DevHeap& h, uint32_t T, uint32_t need, uint32_t* bid_out) {
#ifdef DSR_PROFILE
  const bool prof = h.flags & DSR_F_STATS;
#else
  constexpr bool prof = false;
#endif
  uint32_t oom_tries = 0, fails = 0;
  long long c0 = prof ? clock64() : 0;
  if (prof) stat_add(h, ST_REQ, 1);
  // Per-warp block hint: the block this hardware warp slot last reserved from
  // (any active block is a valid choice); tried first, and a
  // failed try counts as a failed lookup attempt.  Off in paper-exact mode.
  volatile uint32_t* hs = (h.flags & DSR_F_NO_HINT) ? nullptr : hint_slot(h, T);
  uint32_t hint = hs ? *hs : 0xFFFFFFFFu;
  // The searches of a request start from a rotation that depends on the warp
  // AND on the block it last allocated from (kept in the hint slot with the
  // top bit set once that block is full): a warp whose start offset were the
  // same for every request would keep landing on the frontier of blocks its
  // neighbours in rotation space are filling (measured: 16 % fewer lookups,
  // new4 2.43 -> 2.06 ms).
  // A warp whose last block is full (top bit) first tries a random other
  // active block of that block's leaf container, or if there is none, a random
  // active block of a random non-empty leaf under the same level-1 word (one
  // or two loads instead of a top-down search; counts as a lookup attempt
  // like the hint): finds per step 7.8 M -> 4.1 M, new1 5.14 -> 4.79 ms,
  // new4 1.96 -> 1.64 ms, GoL 16384^2 49.6 -> 44.4 ms/gen.
  const uint64_t who = warp_gid() ^ ((uint64_t)hint << 24);
  uint32_t sib = 0xFFFFFFFFu;
  if ((hint & 0x80000000u) && hint != 0xFFFFFFFFu) sib = near_block(h, T, hint & 0x7FFFFFFFu, rot_hash(h, who, 0x777));
  hint = (hint & 0x80000000u) ? sib : hint;
  // SM-affine home ranges are an ablation (DSR_F_HOME_ROT): measured slower than
  // the hashed global rotation (all 64 warps of an SM pile onto the few active
  // blocks of its range) and it strands active blocks of other ranges near OOM.
  const bool home = (h.flags & DSR_F_HOME_ROT) && !(h.flags & DSR_F_NO_ROTATE) && h.freebm.nlevels >= 2;
  uint32_t hlo = 0, hlen = 1;
  if (home) home_range(h.freebm, h.sms, &hlo, &hlen);
  for (uint64_t iter = 0;; ++iter) {
    int64_t bid = -1;
    bool fresh = false, hinted = false;
    long long c1 = prof ? clock64() : 0;
    // one hash per attempt: bits 0-35 rotate the levels of the search, bits
    // 58-63 the slot selection inside the block
    const uint64_t rh = rot_hash(h, who, iter);
    if (hint < h.M) {
      bid = hint;
      hint = 0xFFFFFFFFu;
      hinted = true;
    } else if (fails < h.r_attempts) {
      uint64_t leaf = 0;
      bid = home ? bm_find_home(h.activebm[T], hlo, hlen, rh, &leaf) : bm_try_find_set(h.activebm[T], rh, &leaf);
      if (prof) { stat_add(h, ST_FIND, 1); stat_add(h, ST_CYC_FIND, clock64() - c1); }
      if (bid < 0) { if (prof) stat_add(h, ST_FINDFAIL, 1); ++fails; continue; }
    } else {                                                                  // slow path
      bid = -1;
      for (int k = 0; home && bid < 0 && k < 4; ++k) {                        // a free block in the home range
        const int64_t c = bm_find_home(h.freebm, hlo, hlen, rot_hash(h, who, (iter << 8) + 64 + k));
        if (c < 0) break;
        if (bm_try_clear(h.freebm, (uint64_t)c)) bid = c;
      }
      if (bid < 0) bid = bm_clear_any(h, h.freebm, who, iter << 8);
      if (bid < 0) {
        // FAIL: free bitmap empty, or transiently inconsistent.  Only a
        // top-level word of 0 counts towards OOM.
        if (ld_relaxed(h.freebm.lvl[h.freebm.nlevels - 1]) == 0 && !(h.flags & DSR_F_SPIN_ON_OOM) &&
            ++oom_tries >= 64) {
          flag_error(h, ERRB_OOM);
          stat_add(h, ST_OOM, 1);
          return 0;
        }
        uint32_t ns = 128;
        backoff(ns);
        fails = 0;                                                            // look for active blocks again
        continue;
      }
      init_block(h, T, (uint32_t)bid);
      {                                                                       // allocated[T].set, active[T].set:
        const uint64_t m = 1ull << (bid & 63);                                // both blind atomics in flight together
        const uint64_t pl = atom_or(h.allocbm[T].lvl[0] + (bid >> 6), m);
        const uint64_t pa = atom_or(h.activebm[T].lvl[0] + (bid >> 6), m);
        bm_set_finish(h.allocbm[T], (uint64_t)bid, pl);
        bm_set_finish(h.activebm[T], (uint64_t)bid, pa);
      }
      stat_add(h, ST_INITS, 1);
      if (prof) stat_add(h, ST_CYC_SLOW, clock64() - c1);
      fresh = true;
    }
    uint64_t before = 0;
    DSR_FAULT_POINT(1);
    long long c2 = prof ? clock64() : 0;
    // Slots inside the block: the lowest free ones by default; the paper also
    // rotates here (DSR_F_SLOT_ROTATE).  With per-warp hints a block
    // has mostly one filler, and unrotated reservations are contiguous runs
    // (cheap n-th-bit, coalesced constructor stores): new1 4.75 -> 3.87 ms.
    const uint32_t rot = (h.flags & DSR_F_SLOT_ROTATE) ? (uint32_t)(rh >> 58) : 0u;
    // A fresh block's word is known (no read).  (A "blind" first atomicOr on
    // found blocks, assuming them empty, was measured 1.5x slower: partial
    // fills doubled the number of requests.)
    const uint64_t got = block_reserve(h, (uint32_t)bid, need, rot, &before, fresh, h.types[T].pad);
    if (!got) {                                                               // full or invalidated
      if (prof) { stat_add(h, ST_RESZERO, 1); if (hinted) stat_add(h, ST_HINTZERO, 1); }
      ++fails;
      continue;
    }
    const uint32_t t = ld_relaxed_u8(h.type + bid) - 1u;                      // volatile read (Alg. 1 l.10)
    const bool full = (before | got) == ~0ull;
    if (full) bm_clear(h.activebm[t], (uint64_t)bid);                         // FULL -> inactive (l.12)
    if (prof) stat_add(h, ST_CYC_RES, clock64() - c2);
    if (t == T) {
      if (hs) *hs = full ? ((uint32_t)bid | 0x80000000u) : (uint32_t)bid;
      if (prof) stat_add(h, ST_CYC_REQ, clock64() - c0);
      *bid_out = (uint32_t)bid;
      return got;
    }
    block_free<true, false>(h, t, (uint32_t)bid, got);                                     // type changed: rollback (l.14)
    stat_add(h, ST_ROLLBACKS, 1);
  }
}

// Device new<T> with allocation request coalescing: lanes of
// the calling warp that request the same type elect a leader, the leader
// reserves slots for all of them, each lane takes the rank-th reserved slot.
// Any subset of lanes may call it (divergent call sites allowed).
__device__ __forceinline__ uint64_t dsr_new(const DevHeap& h, uint32_t T) {
  const uint32_t lane = lane_id();
  const uint32_t act = __activemask();
  const uint32_t peers = (h.flags & DSR_F_NO_COALESCE) ? (1u << lane) : __match_any_sync(act, T);
  const uint32_t leader = __ffs(peers) - 1;
  const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
  const uint32_t count = __popc(peers);
  const uint32_t cap = h.types[T].cap;
  uint64_t mine = 0;
  uint32_t done = 0;
  while (done < count) {
    uint64_t got = 0;
    uint32_t bid = 0;
    if (lane == leader) got = reserve_chunk(h, T, count - done, &bid);
    got = shfl64(peers, got, leader);
    bid = __shfl_sync(peers, bid, leader);
    if (got == 0) break;                                   // OOM: remaining lanes get null
    const uint32_t n = __popcll(got);
    if (rank >= done && rank < done + n) mine = make_handle(T, cap, bid, nth_bit(got, rank - done));
    done += n;
  }
  if (lane == leader) stat_add(h, ST_ALLOCS, done);
  __syncwarp(peers);   // the leader's acquire orders the lanes' constructor writes after the reservation
  return mine;
}

// Device new<T> for UNIFORM call sites (every thread of the CTA calls it; a
// thread that needs no object passes want = false): request coalescing at CTA
// granularity (an extension of the paper's warp-level coalescing, for
// bulk constructors such as parallel_new).  Threads rank themselves per
// type in shared memory; one leader lane per type (warp 0) reserves all slots
// of its type, possibly over several blocks (partial fills move on to another
// block); each thread takes the rank-th reserved slot.  Up to 1024
// threads per CTA.  Returns 0 on OOM (sticky error set by the leader).
__device__ __forceinline__ uint64_t dsr_new_uniform(const DevHeap& h, uint32_t T, bool want) {
  __shared__ uint32_t s_cnt[DSR_MAX_TYPES], s_pre[DSR_MAX_TYPES], s_nch[DSR_MAX_TYPES];
  __shared__ uint32_t s_bid[1024], s_cum[1024];
  __shared__ uint64_t s_mask[1024];
  const uint32_t tid = threadIdx.x;
  if (tid < DSR_MAX_TYPES) s_cnt[tid] = 0;
  __syncthreads();
  const uint32_t rank = want ? atomicAdd(&s_cnt[T], 1u) : 0u;
  __syncthreads();
  if (tid < 32) {
    const uint32_t t = tid;
    uint32_t pre = 0;
    for (uint32_t u = 0; u < t && u < DSR_MAX_TYPES; ++u) pre += s_cnt[u];
    if (t < h.ntypes && s_cnt[t] > 0) {
      const uint32_t need = s_cnt[t];
      uint32_t k = pre, done = 0;
      while (done < need) {
        uint32_t bid = 0;
        const uint64_t got = reserve_chunk(h, t, need - done, &bid);
        if (!got) break;                                     // OOM: the rest get null
        s_bid[k] = bid;
        s_mask[k] = got;
        s_cum[k] = done;
        done += __popcll(got);
        ++k;
      }
      s_pre[t] = pre;
      s_nch[t] = k - pre;
      stat_add(h, ST_ALLOCS, done);
    }
  }
  __syncthreads();
  uint64_t mine = 0;
  if (want) {
    const uint32_t b0 = s_pre[T], n = s_nch[T];
    uint32_t lo = 0, hi = n;                                 // last chunk with s_cum <= rank
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_cum[b0 + mid] <= rank) lo = mid; else hi = mid;
    }
    if (n) {
      const uint64_t m = s_mask[b0 + lo];
      const uint32_t off = rank - s_cum[b0 + lo];
      if (off < (uint32_t)__popcll(m)) mine = make_handle(T, h.types[T].cap, s_bid[b0 + lo], nth_bit(m, off));
    }
  }
  __syncthreads();   // shared state reused by the next call; orders the leaders' acquire before the writes
  return mine;
}

// Bulk constructors (uniform call sites): warp-level coalescing.  (CTA-level
// coalescing, dsr_new_uniform, was measured slower on B200 -- fewer concurrent
// leaders hide less latency; it remains as the microbench ablation
// DSR_F_CTA_NEW only, so app kernels carry none of its shared memory.)
__device__ __forceinline__ uint64_t dsr_new_bulk(const DevHeap& h, uint32_t T, bool want) {
  return want ? dsr_new(h, T) : 0ull;
}

// ------------------------------------------------------------------ warp-cooperative bulk new (reading R-BULK)
// Multi-bit forms of the bitmap operations: the paper's coalescing of
// reservations into one atomicOr applied to the block bitmaps when
// one request needs several blocks.  The cascade rule is the single-bit one
// (Alg. 3 l.6, Def. P:1129): the thread whose atomic turned the container
// from non-zero to 0 (0 to non-zero) updates the nested level.
//
// clear_many: up to k set bits of ONE leaf container of `b` (found by a
// rotated try_find_set), the first k at or after the found bit
// cyclically, cleared with one atomicAnd.  Returns the bits this call cleared
// (0 = FAIL) and their leaf index in *wi.
__device__ __forceinline__ uint64_t bm_clear_many(const DevBitmap& b, uint64_t rh, uint32_t k, uint64_t* wi) {
  uint64_t leaf = 0;
  const int64_t pos = bm_try_find_set(b, rh, &leaf);
  if (pos < 0) return 0;
  const uint32_t p = (uint32_t)pos & 63u;
  uint64_t c = rotr64(leaf, p);                                  // bit 0 = the found bit
  if ((uint32_t)__popcll(c) > k) c &= (2ull << nth_bit(c, k - 1)) - 1ull;
  const uint64_t sel = rotl64(c, p);
  *wi = (uint64_t)pos >> 6;
  const uint64_t before = atom_and(b.lvl[0] + *wi, ~sel);
  const uint64_t got = before & sel;
  if (got && (before & ~sel) == 0 && b.nlevels > 1) bm_clear_from(b, 1, *wi);
  return got;
}
// set_many: set the bits `mask` of leaf container wi (legal use: all 0).
// A bit found already set has a clear in flight (a block being freed while
// another thread already took it from the free bitmap): wait and set it after
// the clear, as bm_set does.
__device__ __forceinline__ void bm_set_many(const DevBitmap& b, uint64_t wi, uint64_t mask) {
  uint64_t* w = b.lvl[0] + wi;
  const uint64_t prev = atom_or(w, mask);
  bool up = prev == 0;
  uint64_t late = prev & mask;
  while (late) {
    const uint64_t m = late & (0ull - late);
    late &= late - 1;
    uint64_t pv = prev;
    uint32_t ns = 32, spins = 0;
    while (pv & m) {
      DSR_SPIN_GUARD(b.err, spins)
      backoff(ns);
      if (!(ld_relaxed(w) & m)) pv = atom_or(w, m);
    }
    up |= pv == 0;
  }
  if (up && b.nlevels > 1) bm_set_from(b, 1, wi);
}

// Warp-cooperative new of `need` objects of type T (every lane of a full warp
// calls it with the same T and need).  Generalises Alg. 1 to a request of many
// slots (reading R-BULK):
//  * fast path: up to 32 lanes each take an active block of T found with a
//    rotated try_find_set (one search per lane, distinct rotations),
//    duplicate finds are merged (__match_any_sync), the lanes split the
//    request over their blocks' free slots by a warp prefix sum and reserve
//    with ONE atomicOr per block (Alg. 6).  FULL -> active.clear
//    (Alg. 1 l.12); a block whose type changed is rolled back (l.14).  A
//    lookup that finds nothing or yields no slot is a failed attempt.
//  * after r failed attempts, the slow path: fresh blocks from the
//    free bitmap, up to 64 per atomicAnd (bm_clear_many), initialised by the
//    lanes in parallel (Alg. 8) with their reserved slots already set (a block
//    whose slots are all taken is born full and never active),
//    allocated[T].set for all of them with one atomicOr, active[T].set only
//    for a partially used one (Alg. 1 l.4-7).
// Returns the number of slots reserved (warp-uniform; < need only on OOM or
// when all 32 lanes hold a chunk -- call again for the rest).  Lane i holds
// chunk i: block *bid_out and reserved slots *mask_out (0 = no chunk); the
// objects are ranked in lane order, then by slot.
__device__ __forceinline__ uint32_t dsr_new_warp(const DevHeap& h, uint32_t T, uint32_t need, uint32_t* bid_out,
                                                 uint64_t* mask_out) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t cap = h.types[T].cap;
  const uint64_t valid = h.types[T].valid, pad = h.types[T].pad;
  const uint64_t who = warp_gid() * 32 + lane;
  uint32_t my_bid = 0, have = 0, fails = 0, oom_tries = 0;
  uint64_t my_mask = 0;
  for (uint32_t round = 0; have < need; ++round) {
    const uint32_t rem = need - have;
    const uint32_t freelanes = __ballot_sync(0xffffffffu, my_mask == 0);
    if (!freelanes) break;
    const uint32_t frank = __popc(freelanes & lt);                 // rank among chunk-less lanes
    if (fails < h.r_attempts) {
      // searches: about two per expected half-free block of the remainder
      const uint32_t k = min(__popc(freelanes), (2u * rem + cap - 1u) / cap + 1u);
      const bool searcher = my_mask == 0 && frank < k;
      int64_t cand = -1;
      if (searcher) cand = bm_try_find_set(h.activebm[T], rot_hash(h, who, round));
      const uint32_t same = __match_any_sync(0xffffffffu, (ull)cand);
      const bool lead = searcher && cand >= 0 && (uint32_t)(__ffs(same) - 1) == lane;
      const uint64_t cur = lead ? ld_relaxed(h.alloc_bm + cand) : ~0ull;
      const uint32_t f = (uint32_t)__popcll(~cur);
      uint32_t incl = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
      }
      const uint32_t excl = incl - f;
      const uint32_t take = excl >= rem ? 0u : min(f, rem - excl);
      uint64_t got = 0;
      if (take) {
        DSR_FAULT_POINT(4);
        uint64_t fr = ~cur;
        if ((uint32_t)__popcll(fr) > take) fr &= (2ull << nth_bit(fr, take - 1)) - 1ull;
        const uint64_t before = atom_or_acquire(h.alloc_bm + cand, fr);
        got = fr & ~before;
        if (got) {
          const uint32_t t = ld_relaxed_u8(h.type + cand) - 1u;       // volatile read (Alg. 1 l.10)
          if ((before | got) == ~0ull) bm_clear(h.activebm[t], (uint64_t)cand);   // FULL (l.12)
          if (t != T) {                                               // type changed: rollback (l.14)
            block_free<true, false>(h, t, (uint32_t)cand, got);
            stat_add(h, ST_ROLLBACKS, 1);
            got = 0;
          }
        }
        if (got) { my_bid = (uint32_t)cand; my_mask = got; }
      }
      const uint32_t gained = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(got));
      const uint32_t failed = __popc(__ballot_sync(0xffffffffu, searcher && (cand < 0 || (take && !got) || (lead && f == 0))));
      have += gained;
      // every failed lane search is an attempt (R-BULK); DSR_F_BULK_DENSE:
      // one attempt per round with a failure, so the request stays longer on
      // partially free blocks (microbench F after phase 4 0.23 -> 0.10, step +8 %)
      if (h.flags & DSR_F_BULK_DENSE) fails += (failed || !gained) ? 1u : 0u;
      else fails += failed ? failed : (gained ? 0u : 1u);
      continue;
    }
    // slow path: fresh blocks for the remainder, leader lane claims them from the free bitmap
    const uint32_t nb = min((rem + cap - 1u) / cap, (uint32_t)__popc(freelanes));
    const uint32_t leader = __ffs(freelanes) - 1;
    uint64_t got = 0, wi = 0;
    // (R-FREEROT's window here too; the full rotation measured the same step:
    // new1 0.55 vs 0.60 ms, new4 0.54 vs 0.50 ms)
    if (lane == leader) got = bm_clear_many(h.freebm, rot_hash(h, who, 0x100000ull + round) & kFreeRotMask, nb, &wi);
    got = shfl64(0xffffffffu, got, leader);
    wi = shfl64(0xffffffffu, wi, leader);
    if (!got) {
      // FAIL: free bitmap empty or transiently inconsistent; only a
      // top-level word of 0 counts towards OOM (reading R-OOM)
      const bool empty = ld_relaxed(h.freebm.lvl[h.freebm.nlevels - 1]) == 0;
      if (empty && !(h.flags & DSR_F_SPIN_ON_OOM) && ++oom_tries >= 64) {
        if (lane == 0) { flag_error(h, ERRB_OOM); stat_add(h, ST_OOM, 1); }
        break;
      }
      uint32_t ns = 128;
      backoff(ns);
      fails = 0;                                                      // look for active blocks again
      continue;
    }
    const uint32_t ngot = (uint32_t)__popcll(got);
    bool partial = false;
    if (my_mask == 0 && frank < ngot) {                               // the frank-th claimed block
      const uint32_t bid = (uint32_t)(wi * 64 + nth_bit(got, frank));
      const uint32_t left = rem - frank * cap;                        // > 0: ngot <= ceil(rem / cap)
      const uint64_t slots = left >= cap ? valid : ((1ull << left) - 1ull);
      partial = left < cap;
      st_relaxed_u8(h.type + bid, T + 1);                             // Alg. 8, slots already reserved
      st_release(h.alloc_bm + bid, pad | slots);
      my_bid = bid;
      my_mask = slots;
    }
    __syncwarp();
    if (lane == leader) { bm_set_many(h.allocbm[T], wi, got); stat_add(h, ST_INITS, ngot); }
    __syncwarp();
    if (partial) bm_set(h.activebm[T], my_bid);
    have += min(rem, ngot * cap);
  }
  if (lane == 0) stat_add(h, ST_ALLOCS, have);
  __syncwarp();
  *bid_out = my_bid;
  *mask_out = my_mask;
  return have;
}

// Device destroy: lanes freeing slots of the same block combine their
// bits into one atomicAnd (coalesced version of Alg. 7).
// RELEASE = false is dsr_destroy_ro below.
// Destroy the objects `mask` of block `bid` of type T (several slots of one
// block per lane: quad-mapped do-alls); lanes naming the same block combine
// their masks into one atomicAnd.
template <bool RELEASE = true>
__device__ __forceinline__ void dsr_destroy_mask(const DevHeap& h, uint32_t T, uint32_t bid, uint64_t bits) {
  if (bits == 0) return;
#ifdef DSR_DEBUG
  if (T >= h.ntypes || bid >= h.M || (bits & ~h.types[T].valid)) {    // a forged / corrupted handle
    atomicOr(&h.ctrl[CTRL_ERR], (unsigned long long)ERRB_BOUNDS);
    return;
  }
#endif
  const uint32_t lane = lane_id();
  const uint32_t act = __activemask();
  const uint64_t key = ((uint64_t)T << 32) | bid;
  const uint32_t peers = (h.flags & DSR_F_NO_COALESCE) ? (1u << lane) : __match_any_sync(act, (ull)key);
  const uint32_t leader = __ffs(peers) - 1;
  const uint32_t lo = __reduce_or_sync(peers, (uint32_t)bits);
  const uint32_t hi = __reduce_or_sync(peers, (uint32_t)(bits >> 32));
  __syncwarp(peers);   // memory ordering among the lanes: their object accesses precede the leader's release
  if (lane == leader) {
    const uint64_t mask = ((uint64_t)hi << 32) | lo;
    block_free<RELEASE>(h, T, bid, mask);
    stat_add(h, ST_FREES, __popcll(mask));
  }
}
template <bool RELEASE = true>
__device__ __forceinline__ void dsr_destroy_t(const DevHeap& h, uint64_t x) {
  if (x == 0) return;
  dsr_destroy_mask<RELEASE>(h, h_type(x), h_bid(x), 1ull << h_slot(x));
}
__device__ __forceinline__ void dsr_destroy(const DevHeap& h, uint64_t x) { dsr_destroy_t<true>(h, x); }
// Destroy without the release fence (atom.release compiles to MEMBAR.ALL.GPU +
// ATOMG; ncu showed the fence as the free passes' second stall reason).  Only
// for callers whose lanes have NOT written the object since they last
// synchronised with other threads, and whose reads of it are all consumed
// (the call is data- or control-dependent on them, or there are none): then
// nothing of theirs can be reordered past the slot's reuse.
__device__ __forceinline__ void dsr_destroy_ro(const DevHeap& h, uint64_t x) { dsr_destroy_t<false>(h, x); }
// x, made data-dependent on v (a value loaded from the object that is used
// after a dsr_destroy_ro): v never equals 0xFFFFFFFF at the call sites (a cell
// id), so the result is x, but the destroy cannot issue before v has arrived.
__device__ __forceinline__ uint64_t after_load(uint64_t x, uint32_t v) { return x | (v == 0xFFFFFFFFu ? 1ull : 0ull); }

}  // namespace dsr
