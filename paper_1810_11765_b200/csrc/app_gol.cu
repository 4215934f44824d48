// app_gol.cu -- Game of Life with O(#alive) work (Table 1; reading
// R-GOL).  Types: 0 = Alive{cell u32, is_new u8, action u8},
// 1 = Candidate{cell u32, action u8}.  The static cell grid `cell[c]` holds
// the handle of the object at c (0 = empty); liveness of a neighbour is read
// from the handle's type bits, never from the object ("fast
// instance-of checks").  Four do-alls per generation (Table 1):
//   1 Candidate.prepare  2 Alive.prepare  3 Candidate.update  4 Alive.update
// In pass 4 a new Alive creates a Candidate on every empty neighbour exactly
// once: the creator claims the empty cell with atomicCAS(0 -> RESERVED), so
// the created set is the same for every visit order.
#include <cuda.h>   // cuStreamWaitValue32 (types only: resolved at run time, no libcuda link dependency)
#include "dsr_host.h"

namespace dsr {

enum { GOL_ALIVE = 0, GOL_CAND = 1 };
enum { ACT_NONE = 0, ACT_SPAWN = 1, ACT_DIE = 2 };
constexpr uint64_t kReserved = 1;   // not a handle: type bits 0

__device__ __forceinline__ uint32_t gol_nbr(uint32_t W, uint32_t H, uint32_t c, int k, uint32_t ghost = 0) {
  // Moore neighbourhood, k = 0..7 (row-major order of offsets); x wraps; y wraps
  // on the W x H torus, or (sharded, ghost rows 0 and H + 1) never leaves rows 0..H+1
  const uint32_t x = c % W, y = c / W;
  const int dx = (k < 3) ? k - 1 : (k == 3 ? -1 : (k == 4 ? 1 : k - 6));
  const int dy = (k < 3) ? -1 : (k < 5 ? 0 : 1);
  const uint32_t nx = dx < 0 ? (x == 0 ? W - 1 : x - 1) : (dx > 0 ? (x + 1 == W ? 0 : x + 1) : x);
  const uint32_t ny = ghost ? (uint32_t)((int)y + dy)
                            : (dy < 0 ? (y == 0 ? H - 1 : y - 1) : (dy > 0 ? (y + 1 == H ? 0 : y + 1) : y));
  return ny * W + nx;
}
__device__ __forceinline__ bool gol_local(const dsr_gol_args& a, uint32_t c) {
  const uint32_t y = c / a.W;
  return !a.ghost || (y >= 1 && y <= a.H);
}
// a ghost cell holding a neighbour shard's alive cell: a handle value whose
// type bits say Alive, never dereferenced
__device__ __forceinline__ uint64_t ghost_alive(const DevHeap& h) { return make_handle(GOL_ALIVE, h.types[GOL_ALIVE].cap, 0, 0); }

// ---- optional alive-bit mirror (a.bits): 1 bit per cell, row pitch ceil(W/32) words
__device__ __forceinline__ uint32_t gol_pitch(const dsr_gol_args& a) { return (a.W + 31) >> 5; }
__device__ __forceinline__ void gol_bit_set(const dsr_gol_args& a, uint32_t c, bool v) {
  const uint32_t x = c % a.W, y = c / a.W;
  uint32_t* w = a.bits + (size_t)y * gol_pitch(a) + (x >> 5);
  const uint32_t m = 1u << (x & 31);
  if (v) atomicOr(w, m); else atomicAnd(w, ~m);
}
__device__ __forceinline__ uint32_t gol_bit(const uint32_t* row, uint32_t x) {
  return (__ldg(row + (x >> 5)) >> (x & 31)) & 1u;
}
// alive cells among x-1, x, x+1 (torus in x) of one row
__device__ __forceinline__ uint32_t gol_row3(const dsr_gol_args& a, const uint32_t* row, uint32_t x) {
  const uint32_t o = x & 31;
  if (o != 0 && o != 31 && x + 1 < a.W) return __popc((__ldg(row + (x >> 5)) >> (o - 1)) & 7u);
  const uint32_t xl = x == 0 ? a.W - 1 : x - 1, xr = x + 1 == a.W ? 0 : x + 1;
  return gol_bit(row, xl) + gol_bit(row, x) + gol_bit(row, xr);
}
__device__ __forceinline__ uint32_t gol_alive_nbrs_bits(const dsr_gol_args& a, uint32_t c) {
  const uint32_t x = c % a.W, y = c / a.W, P = gol_pitch(a);
  const uint32_t ym = a.ghost ? y - 1 : (y == 0 ? a.H - 1 : y - 1);
  const uint32_t yp = a.ghost ? y + 1 : (y + 1 == a.H ? 0 : y + 1);
  const uint32_t* r = a.bits + (size_t)y * P;
  return gol_row3(a, a.bits + (size_t)ym * P, x) + gol_row3(a, r, x) + gol_row3(a, a.bits + (size_t)yp * P, x) -
         gol_bit(r, x);
}

__device__ __forceinline__ uint32_t gol_alive_nbrs(const dsr_gol_args& a, uint32_t c) {
  if (a.bits) return gol_alive_nbrs_bits(a, c);
  uint32_t k = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d)
    k += h_is(__ldg((const unsigned long long*)a.cell + gol_nbr(a.W, a.H, c, d, a.ghost)), GOL_ALIVE);
  return k;
}

__device__ __forceinline__ uint64_t new_alive(const DevHeap& h, uint32_t c, uint8_t is_new) {
  const uint64_t nh = dsr_new(h, GOL_ALIVE);
  if (nh) {
    *field_ptr<uint32_t>(h, nh, 0) = c;
    *field_ptr<uint8_t>(h, nh, 1) = is_new;
    *field_ptr<uint8_t>(h, nh, 2) = ACT_NONE;
  }
  return nh;
}
__device__ __forceinline__ uint64_t new_cand(const DevHeap& h, uint32_t c) {
  const uint64_t nh = dsr_new(h, GOL_CAND);
  if (nh) {
    *field_ptr<uint32_t>(h, nh, 0) = c;
    *field_ptr<uint8_t>(h, nh, 1) = ACT_NONE;
  }
  return nh;
}

// ---- initial state: Alive for alive cells, Candidate for dead cells with an alive neighbour
__global__ void __launch_bounds__(256) k_gol_init(DevHeap h, uint64_t n, dsr_gol_args a, int cand) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    const uint32_t c = (uint32_t)i;
    bool want = false;
    if (i < n && !cand && a.bits && a.alive0[c]) gol_bit_set(a, c, true);
    if (i < n && !gol_local(a, c)) {
      if (!cand) a.cell[c] = a.alive0[c] ? ghost_alive(h) : 0ull;   // ghost rows: neighbours' alive cells
    } else if (i < n) {
      const bool alive = a.alive0[c];
      if (!cand) {
        want = alive;
      } else if (!alive) {
        for (int d = 0; d < 8; ++d) want |= a.alive0[gol_nbr(a.W, a.H, c, d, a.ghost)] != 0;
      }
    }
    const uint32_t T = cand ? GOL_CAND : GOL_ALIVE;
    const uint64_t nh = dsr_new_bulk(h, T, want);
    if (nh) {
      *field_ptr<uint32_t>(h, nh, 0) = c;
      if (!cand) {
        *field_ptr<uint8_t>(h, nh, 1) = 0;
        *field_ptr<uint8_t>(h, nh, 2) = ACT_NONE;
      } else {
        *field_ptr<uint8_t>(h, nh, 1) = ACT_NONE;
      }
    }
    if (want) a.cell[c] = nh;
  }
}

// Alive.prepare's stores: is_new = 0, action = DIE iff k < 2 or k > 3.  Every
// Alive enters pass 2 with action NONE (created with NONE; pass 4 destroys the
// old ones marked DIE, and a new one is created after pass 2), and is_new is
// 1 only for the Alives pass 3 created: the stores are made only where they
// change the byte (a store of an unchanged byte still dirties its sector).
__device__ __forceinline__ void gol_alive_prepare_store(const DevHeap& h, uint64_t hd, uint32_t k) {
  uint8_t* const is_new = field_ptr<uint8_t>(h, hd, 1);
  if (*is_new) *is_new = 0;
  if (k < 2 || k > 3) *field_ptr<uint8_t>(h, hd, 2) = ACT_DIE;
}

struct GolCandPrepare {   // pass 1
  typedef dsr_gol_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    const uint32_t k = gol_alive_nbrs(a, c);
    // every Candidate enters pass 1 with action NONE (created with NONE; pass 3
    // destroys the ones whose action is not NONE), so NONE needs no store
    if (k == 3 || k == 0) *field_ptr<uint8_t>(h, T, 1, b, s) = k == 3 ? ACT_SPAWN : ACT_DIE;
  }
};
struct GolAlivePrepare {  // pass 2
  typedef dsr_gol_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    const uint32_t k = gol_alive_nbrs(a, c);
    gol_alive_prepare_store(h, make_handle(T, h.types[T].cap, b, s), k);
  }
};
struct GolCandUpdate {    // pass 3 (allocates Alive)
  typedef dsr_gol_args Args;
  DSR_NO_ACC
  // k_doall_sel: only Candidates with an action do work
  static __device__ __forceinline__ bool select(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args&) {
    return *field_ptr<uint8_t>(h, T, 1, b, s) != ACT_NONE;
  }
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint8_t act = *field_ptr<uint8_t>(h, T, 1, b, s);
    if (act == ACT_NONE) return;
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    // never written; act is consumed by the branch, c by the handle (after_load)
    dsr_destroy_ro(h, after_load(make_handle(T, h.types[T].cap, b, s), c));
    if (act == ACT_SPAWN) a.cell[c] = new_alive(h, c, 1);
    else a.cell[c] = 0;
    if (act == ACT_SPAWN && a.bits) gol_bit_set(a, c, true);
  }
};
struct GolAliveUpdate {   // pass 4 (allocates Candidate)
  typedef dsr_gol_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    uint32_t todo = 0;                                   // bit d: create a Candidate at neighbour d; bit 8: at c
    if (*field_ptr<uint8_t>(h, T, 1, b, s)) {            // new Alive: claim the empty neighbours
      // the 8 neighbour loads first (independent, all in flight), then a CAS
      // only on the cells that read empty
      uint64_t nb[8];
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const uint32_t e = gol_nbr(a.W, a.H, c, d, a.ghost);
        nb[d] = gol_local(a, e) ? ld_relaxed((const uint64_t*)a.cell + e) : 1ull;   // a neighbour shard's cell: its owner creates it
      }
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        if (nb[d] != 0) continue;
        unsigned long long* pe = (unsigned long long*)a.cell + gol_nbr(a.W, a.H, c, d, a.ghost);
        if (atomicCAS(pe, 0ull, kReserved) == 0ull) todo |= 1u << d;
      }
    } else if (*field_ptr<uint8_t>(h, T, 2, b, s) == ACT_DIE) {
      dsr_destroy_ro(h, after_load(make_handle(T, h.types[T].cap, b, s), c));   // read-only, c consumed
      if (a.bits) gol_bit_set(a, c, false);
      todo = 1u << 8;
    }
    // allocate in warp-synchronous rounds so that every lane's k-th Candidate
    // is requested together (one coalesced request per round)
    const uint32_t rounds = __reduce_max_sync(__activemask(), (uint32_t)__popc(todo));
    for (uint32_t r = 0; r < rounds; ++r) {
      if (todo) {
        const int d = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t e = d == 8 ? c : gol_nbr(a.W, a.H, c, d, a.ghost);
        a.cell[e] = new_cand(h, e);
      }
    }
  }
};

// ---- row sharding: one exchange of boundary masks per generation
__device__ __forceinline__ uint8_t gol_mask(const DevHeap& h, uint64_t hd) {
  if (!h_is(hd, GOL_ALIVE)) return 0;
  const uint8_t is_new = *field_ptr<uint8_t>(h, hd, 1), act = *field_ptr<uint8_t>(h, hd, 2);
  const bool next_alive = is_new || act != ACT_DIE;          // survives pass 4
  return (uint8_t)((next_alive ? 1u : 0u) | (is_new ? 2u : 0u));
}
// after pass 3: next-alive / new-alive bits of my first and last local row
__global__ void k_gol_halo_pack(DevHeap h, uint64_t n, dsr_gol_args a) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    a.halo[x] = gol_mask(h, a.cell[(uint64_t)1 * a.W + x]);
    a.halo[a.W + x] = gol_mask(h, a.cell[(uint64_t)a.H * a.W + x]);
  }
}
// Peer-memory exchange (fused pack + send): after pass 3, one CTA computes
// the masks of my row 1 and row H and stores them straight into the halo
// buffers of the shards above / below (their segment "from below" / "from
// above" of this generation's parity), then -- all stores issued, fenced at
// system scope -- sets their flags to gen + 1 with a system-scope release.
// Over NVLink the stores are the transfer; there is no staging copy and no
// collective call.
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(1024) k_gol_halo_push(DevHeap h, dsr_gol_args a) {
  const uint32_t W = a.W, par = a.gen & 1u;
  uint8_t* const to_up = a.peer_up + (size_t)(3u + 2u * par) * W;       // the upper shard's "from below"
  uint8_t* const to_down = a.peer_down + (size_t)(2u + 2u * par) * W;   // the lower shard's "from above"
  for (uint32_t x = threadIdx.x; x < W; x += blockDim.x) {
    to_up[x] = gol_mask(h, a.cell[(uint64_t)1 * W + x]);
    to_down[x] = gol_mask(h, a.cell[(uint64_t)a.H * W + x]);
  }
  __threadfence_system();                                              // every thread's stores, system scope,
  __syncthreads();                                                     // before the flags
  if (threadIdx.x == 0) {
    st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer_up + DSR_GOL_PEER_FLAGS(W)) + 1, a.gen + 1u);
    st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer_down + DSR_GOL_PEER_FLAGS(W)), a.gen + 1u);
  }
}

// before pass 4: ghost rows := the neighbours' next-alive cells (read by the
// next generation's prepare passes), and a Candidate on every empty boundary
// cell next to a remote new Alive (the owner computes it; the CAS claim makes
// it exactly once together with pass 4's local claims)
__global__ void __launch_bounds__(256) k_gol_halo_apply(DevHeap h, uint64_t n, dsr_gol_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t in0 = 2, in1 = 3;                                           // received segments (pack + collective)
  if (a.peer_up) {
    // peer mode: the launching stream waited (cuStreamWaitValue32) until both
    // neighbours' flags reached gen + 1; the acquire loads order this kernel's
    // reads of their masks after those flags (they pass at once)
    if (threadIdx.x == 0) {
      const uint32_t* f = reinterpret_cast<const uint32_t*>(a.halo + DSR_GOL_PEER_FLAGS(a.W));
      uint32_t ns = 64;
      while (ld_acquire_sys_u32(f) < a.gen + 1u || ld_acquire_sys_u32(f + 1) < a.gen + 1u) {
        __nanosleep(ns);
        ns = ns < 1024 ? ns * 2 : 1024;
      }
    }
    __syncthreads();
    in0 = 2u + 2u * (a.gen & 1u);
    in1 = 3u + 2u * (a.gen & 1u);
  }
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < 2 * n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    bool want = false;
    uint32_t e = 0;
    if (i < 2 * n) {
      const uint32_t side = (uint32_t)(i / n), x = (uint32_t)(i % n);
      const uint8_t* m = a.halo + (size_t)(side ? in1 : in0) * a.W;   // received masks
      const uint32_t grow = side ? a.H + 1 : 0, brow = side ? a.H : 1;   // ghost row, my boundary row
      a.cell[(uint64_t)grow * a.W + x] = (m[x] & 1) ? ghost_alive(h) : 0ull;
      if (a.bits) gol_bit_set(a, grow * a.W + x, m[x] & 1);
      const uint32_t xl = x == 0 ? a.W - 1 : x - 1, xr = x + 1 == a.W ? 0 : x + 1;
      if ((m[xl] | m[x] | m[xr]) & 2) {
        e = brow * a.W + x;
        unsigned long long* pe = (unsigned long long*)a.cell + e;
        want = ld_relaxed((const uint64_t*)pe) == 0 && atomicCAS(pe, 0ull, kReserved) == 0ull;
      }
    }
    const uint64_t nh = dsr_new_bulk(h, GOL_CAND, want);
    if (nh) {
      *field_ptr<uint32_t>(h, nh, 0) = e;
      *field_ptr<uint8_t>(h, nh, 1) = ACT_NONE;
    }
    if (want) a.cell[e] = nh;
  }
}
struct GolDump {
  typedef dsr_gol_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    uint32_t v;
    if (T == GOL_ALIVE) v = 1u | ((uint32_t)*field_ptr<uint8_t>(h, T, 1, b, s) << 8) | ((uint32_t)*field_ptr<uint8_t>(h, T, 2, b, s) << 16);
    else v = 2u | ((uint32_t)*field_ptr<uint8_t>(h, T, 1, b, s) << 16);
    a.dump[c] = v;
  }
};

// ---- cell-tiled do-alls (the same four methods, enumerated through the cell
// grid instead of the block list).
// Every Alive / Candidate sits in exactly one cell, so visiting the cells
// whose handle has the pass's type visits every object of that type exactly
// once; objects a pass creates are placed in cells by the thread that owns
// the cell after its visit, or in cells whose new content is not of the
// pass's type (Candidates in pass 4), so none is visited by the pass that
// creates it.
// Prepare passes: a CTA stages an (8 + 2) x (128 + 2) tile of handles (8-B,
// coalesced row segments) in shared memory and counts each cell's alive
// neighbours from it (P:333 type bits); the object's action is written
// through its handle.  Update passes: one thread per cell in row-major order,
// so the objects a warp creates (new Alives in pass 3, Candidates in pass 4)
// come from 32 neighbouring cells and go into one block (coalesced request,
// P:649): blocks stay spatially coherent across generations.
constexpr int kTileH = 8, kTileW = 128;
template <int PASS>
__global__ void __launch_bounds__(256) k_gol_tile_prepare(DevHeap h, dsr_gol_args a) {
  __shared__ unsigned long long s[kTileH + 2][kTileW + 2];
  const uint32_t W = a.W, H = a.H, row0 = a.ghost ? 1u : 0u;
  const uint32_t rows_total = a.ghost ? H + 2 : H;
  const uint32_t tx = (W + kTileW - 1) / kTileW, ty = (H + kTileH - 1) / kTileH;
  const uint32_t T = PASS == 1 ? GOL_CAND : GOL_ALIVE;
  const uint32_t nt = tx * ty, t0 = (uint32_t)((uint64_t)blockIdx.x * nt / gridDim.x),
                 t1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nt / gridDim.x);
  for (uint32_t tile = t0; tile < t1; ++tile) {                             // blocked: neighbouring tiles per CTA
    const uint32_t y0 = (tile / tx) * kTileH, x0 = (tile % tx) * kTileW;   // local cell coordinates
    __syncthreads();                                                        // the previous tile is consumed
    for (uint32_t i = threadIdx.x; i < (kTileH + 2) * (kTileW + 2); i += blockDim.x) {
      const int r = (int)(i / (kTileW + 2)), cc = (int)(i % (kTileW + 2));
      const int yy = (int)y0 + r - 1, xx = (int)x0 + cc - 1;               // local row -1 .. H + 7
      int gy = a.ghost ? yy + 1 : ((yy % (int)H) + (int)H) % (int)H;       // grid row (ghost rows 0, H + 1)
      const uint32_t gx = (uint32_t)(((xx % (int)W) + (int)W) % (int)W);
      s[r][cc] = (gy >= 0 && gy < (int)rows_total) ? __ldg((const unsigned long long*)a.cell + (size_t)gy * W + gx)
                                                   : 0ull;
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < kTileH * kTileW; idx += blockDim.x) {
      const uint32_t r = idx / kTileW, cc = idx % kTileW, y = y0 + r, x = x0 + cc;
      if (y >= H || x >= W) continue;
      const uint64_t hd = s[r + 1][cc + 1];
      if (!h_is(hd, T)) continue;
      uint32_t k = 0;
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
          if (dy != 1 || dx != 1) k += h_is(s[r + dy][cc + dx], GOL_ALIVE);
      if (PASS == 1) {
        if (k == 3 || k == 0) *field_ptr<uint8_t>(h, hd, 1) = k == 3 ? ACT_SPAWN : ACT_DIE;   // NONE: unchanged
      } else {
        gol_alive_prepare_store(h, hd, k);
      }
    }
    (void)row0;
  }
}
// Update passes: warp-level, no CTA barriers.  Each warp owns one contiguous
// run of 256-cell chunks (blocked over all warps of the grid, so a warp's
// allocations -- its hint block, P:649 -- fill with objects of neighbouring
// cells and blocks stay spatially coherent across generations).  Per chunk
// the warp loads the 256 handles (8 coalesced rows of 32), compacts those of
// the pass's type into its shared-memory list with ballots (row-major order),
// and runs the method over the list with full warps: lane j gets the j-th of
// 32 neighbouring objects, so destroys and news coalesce per block.  (The
// previous CTA-wide compaction of 2048-cell chunks needed four barriers per
// chunk and left the allocation latency exposed.)
constexpr int kUpdChunk = 256;
#ifndef DSR_GOL_UPD_MINB
#define DSR_GOL_UPD_MINB 4
#endif
template <int PASS>
__global__ void __launch_bounds__(256, DSR_GOL_UPD_MINB) k_gol_tile_update(DevHeap h, dsr_gol_args a) {
  __shared__ unsigned long long s_hd[8][kUpdChunk];
  const uint32_t W = a.W, row0 = a.ghost ? 1u : 0u;
  const uint64_t n = (uint64_t)W * a.H;
  const uint32_t T = PASS == 3 ? GOL_CAND : GOL_ALIVE;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long* const lst = s_hd[wid];
  NoAcc acc;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5, gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nch = (n + kUpdChunk - 1) / kUpdChunk;
  const uint64_t c0 = gw * nch / nw, c1 = (gw + 1) * nch / nw;
  const unsigned long long* cells = (const unsigned long long*)a.cell + (uint64_t)row0 * W;
  for (uint64_t ch = c0; ch < c1; ++ch) {
    const uint64_t base = ch * kUpdChunk;
    unsigned long long v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t i = base + k * 32 + lane;
      v[k] = i < n ? ld_relaxed((const uint64_t*)cells + i) : 0ull;
    }
    uint32_t pos = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool m = h_is(v[k], T);
      const uint32_t bal = __ballot_sync(0xffffffffu, m);
      if (m) lst[pos + __popc(bal & ((1u << lane) - 1u))] = v[k];
      pos += __popc(bal);
    }
    __syncwarp();
    for (uint32_t j = lane; j < pos; j += 32) {
      const uint64_t hd = lst[j];
      if (PASS == 3) GolCandUpdate::run(h, T, h_bid(hd), h_slot(hd), a, acc);
      else GolAliveUpdate::run(h, T, h_bid(hd), h_slot(hd), a, acc);
    }
    __syncwarp();                                                      // lst consumed before the next chunk
  }
}

bool gol_method_info(uint32_t id, MethodInfo* mi) {
  switch (id) {
    case DSR_M_GOL_CAND_PREPARE_TILED: case DSR_M_GOL_ALIVE_PREPARE_TILED: case DSR_M_GOL_CAND_UPDATE_TILED:
    case DSR_M_GOL_ALIVE_UPDATE_TILED:
      *mi = {4, sizeof(dsr_gol_args)}; return true;      // enumerated through the cell grid: no block list
    case DSR_M_GOL_CAND_PREPARE: case DSR_M_GOL_ALIVE_PREPARE: case DSR_M_GOL_DUMP:
      *mi = {0, sizeof(dsr_gol_args)}; return true;
    case DSR_M_GOL_CAND_UPDATE:
      *mi = {1, sizeof(dsr_gol_args)}; return true;
    case DSR_M_GOL_ALIVE_UPDATE:                        // up to 8 new Candidates per visit: dynamic
      *mi = {2, sizeof(dsr_gol_args)}; return true;
  }
  return false;
}

bool gol_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  switch (id) {
    case DSR_M_GOL_CAND_PREPARE: launch_doall<GolCandPrepare>(c, T, snapshot, args); return true;
    case DSR_M_GOL_ALIVE_PREPARE: launch_doall<GolAlivePrepare>(c, T, snapshot, args); return true;
    // Candidate.update as a selective do-all (k_doall_sel: the Candidates with
    // an action in full warps): 6.5 -> 4.5 ms at 16384^2.  Alive.update
    // selective was slower (7.7 -> 10.7 ms: with 32 newborns per warp the
    // rounds of Candidate creation run to the warp's maximum of up to 8), so
    // it keeps the dynamic element loop.
#ifdef DSR_GOL_NO_SEL
    case DSR_M_GOL_CAND_UPDATE: launch_doall<GolCandUpdate>(c, T, snapshot, args); return true;
#else
    case DSR_M_GOL_CAND_UPDATE: launch_doall_sel<GolCandUpdate>(c, T, args); return true;
#endif
    case DSR_M_GOL_ALIVE_UPDATE: launch_doall<GolAliveUpdate>(c, T, snapshot, args); return true;
    case DSR_M_GOL_DUMP: launch_doall<GolDump>(c, T, snapshot, args); return true;
    case DSR_M_GOL_CAND_PREPARE_TILED: case DSR_M_GOL_ALIVE_PREPARE_TILED:
    case DSR_M_GOL_CAND_UPDATE_TILED: case DSR_M_GOL_ALIVE_UPDATE_TILED: {
      const dsr_gol_args a = *(const dsr_gol_args*)args;
      if (a.bits || a.W < 3 || a.H < 1) return false;
      const bool cand = id == DSR_M_GOL_CAND_PREPARE_TILED || id == DSR_M_GOL_CAND_UPDATE_TILED;
      if (T != (cand ? (uint32_t)GOL_CAND : (uint32_t)GOL_ALIVE) || c.rk >= 0) return false;
      if (id == DSR_M_GOL_CAND_PREPARE_TILED)
        k_gol_tile_prepare<1><<<persistent_grid(c, k_gol_tile_prepare<1>), 256, 0, c.st>>>(c.h, a);
      else if (id == DSR_M_GOL_ALIVE_PREPARE_TILED)
        k_gol_tile_prepare<2><<<persistent_grid(c, k_gol_tile_prepare<2>), 256, 0, c.st>>>(c.h, a);
      else if (id == DSR_M_GOL_CAND_UPDATE_TILED)
        k_gol_tile_update<3><<<persistent_grid(c, k_gol_tile_update<3>), 256, 0, c.st>>>(c.h, a);
      else
        k_gol_tile_update<4><<<persistent_grid(c, k_gol_tile_update<4>), 256, 0, c.st>>>(c.h, a);
      count_launch();
      return true;
    }
  }
  return false;
}

bool gol_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_K_GOL_INIT_ALIVE && id != DSR_K_GOL_INIT_CAND && id != DSR_K_GOL_HALO_PACK &&
      id != DSR_K_GOL_HALO_APPLY && id != DSR_K_GOL_HALO_PUSH)
    return false;
  if (bytes != sizeof(dsr_gol_args) || c.h.ntypes < 2) { *ok = 0; return true; }
  const dsr_gol_args a = *(const dsr_gol_args*)args;
  if (id == DSR_K_GOL_HALO_PUSH) {
    if (!a.ghost || !a.halo || !a.peer_up || !a.peer_down || n != a.W) { *ok = 0; return true; }
    k_gol_halo_push<<<1, 1024, 0, c.st>>>(c.h, a);
    count_launch();
    return true;
  }
  if (id == DSR_K_GOL_HALO_PACK || id == DSR_K_GOL_HALO_APPLY) {
    if (!a.ghost || !a.halo || n != a.W) { *ok = 0; return true; }
    if (id == DSR_K_GOL_HALO_APPLY && a.peer_up) {
      // the wait for the neighbours' pushes is a stream-level wait on the flags
      // (front end, no SM held): their kernels -- on other GPUs, or other
      // processes time-sharing this one -- run meanwhile
      typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
      static WaitFn wait = nullptr;
      if (!wait) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
          *ok = 0;
          return true;
        }
        wait = (WaitFn)fn;
      }
      const CUdeviceptr f = (CUdeviceptr)(a.halo + DSR_GOL_PEER_FLAGS(a.W));
      if (wait((CUstream)c.st, f, a.gen + 1u, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS ||
          wait((CUstream)c.st, f + 4, a.gen + 1u, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
        *ok = 0;
        return true;
      }
    }
    if (id == DSR_K_GOL_HALO_PACK) k_gol_halo_pack<<<grid_for(c, n, k_gol_halo_pack), 256, 0, c.st>>>(c.h, n, a);
    else k_gol_halo_apply<<<grid_for(c, 2 * n, k_gol_halo_apply), 256, 0, c.st>>>(c.h, n, a);
    count_launch();
    return true;
  }
  if ((uint64_t)a.W * (a.H + (a.ghost ? 2 : 0)) != n) { *ok = 0; return true; }
  k_gol_init<<<grid_for(c, n, k_gol_init), 256, 0, c.st>>>(c.h, n, a, id == DSR_K_GOL_INIT_CAND);
  count_launch();
  return true;
}

// ---- static-allocation baseline: Life on a u8 cell grid, no objects
__global__ void __launch_bounds__(256) k_gol_static(uint32_t W, uint32_t H, const uint8_t* cur, uint8_t* next) {
  __shared__ uint8_t s[kTileH + 2][kTileW + 2];
  const uint32_t tx = (W + kTileW - 1) / kTileW, ty = (H + kTileH - 1) / kTileH;
  for (uint32_t tile = blockIdx.x; tile < tx * ty; tile += gridDim.x) {
    const uint32_t y0 = (tile / tx) * kTileH, x0 = (tile % tx) * kTileW;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < (kTileH + 2) * (kTileW + 2); i += blockDim.x) {
      const int r = (int)(i / (kTileW + 2)), cc = (int)(i % (kTileW + 2));
      const uint32_t gy = (uint32_t)((((int)y0 + r - 1) % (int)H + (int)H) % (int)H);
      const uint32_t gx = (uint32_t)((((int)x0 + cc - 1) % (int)W + (int)W) % (int)W);
      s[r][cc] = __ldg(cur + (size_t)gy * W + gx);
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < kTileH * kTileW; idx += blockDim.x) {
      const uint32_t r = idx / kTileW, cc = idx % kTileW, y = y0 + r, x = x0 + cc;
      if (y >= H || x >= W) continue;
      const uint32_t k = s[r][cc] + s[r][cc + 1] + s[r][cc + 2] + s[r + 1][cc] + s[r + 1][cc + 2] + s[r + 2][cc] +
                         s[r + 2][cc + 1] + s[r + 2][cc + 2];
      next[(size_t)y * W + x] = (k == 3 || (k == 2 && s[r + 1][cc + 1])) ? 1 : 0;
    }
  }
}

}  // namespace dsr

extern "C" dsr_status dsr_gol_static_step(const dsr_gol_static_args* a, uint32_t steps, void* stream) {
  using namespace dsr;
  if (!a || !a->cur || !a->next || a->W < 3 || a->H < 3) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return DSR_ERR_CUDA;
  const uint64_t tiles = (uint64_t)((a->W + kTileW - 1) / kTileW) * ((a->H + kTileH - 1) / kTileH);
  const int g = (int)(tiles < (uint64_t)sms * 8 ? tiles : (uint64_t)sms * 8);
  uint8_t *c = a->cur, *n = a->next;
  for (uint32_t k = 0; k < steps; ++k) {
    k_gol_static<<<g, 256, 0, st>>>(a->W, a->H, c, n);
    count_launch();
    uint8_t* t = c; c = n; n = t;
  }
  if (c != a->cur && cudaMemcpyAsync(a->cur, c, (size_t)a->W * a->H, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return DSR_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? DSR_OK : DSR_ERR_CUDA;
}
