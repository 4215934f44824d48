// app_wator.cu -- Wa-Tor predator-prey (Table 1; reading R-WATOR).
// Types: 0 = Fish{cell, target, egg: u32}, 1 = Shark{cell, target, egg, energy: u32},
// 2 = Cell{id u32, agent u64, req[5] u8}.  Cells are heap objects created by
// parallel_new in id order; cells[id] maps an id to its handle.
// Eight do-alls per step (Table 1): Cell.prepare, Fish.prepare, Cell.decide,
// Fish.update, Cell.prepare, Shark.prepare, Cell.decide, Shark.update.
// Conflicts are resolved by the target cell (request / decide), so every
// field has one writer per pass and the result does not depend on the order
// in which objects are visited; randomness is key(seed, step, phase, cell).
#include "dsr_host.h"

namespace dsr {

enum { WT_FISH = 0, WT_SHARK = 1, WT_CELL = 2 };
enum { PH_FISH_REQ = 1, PH_FISH_DEC = 2, PH_SHARK_REQ = 3, PH_SHARK_DEC = 4 };

__device__ __forceinline__ uint32_t wt_nbr(uint32_t W, uint32_t H, uint32_t c, uint32_t d, uint32_t ghost = 0) {
  // von Neumann neighbour d in {N, E, S, W} on the torus; sharded (ghost rows
  // 0 and H + 1): no wrap in y, a boundary row's N/S neighbour is a ghost cell
  const uint32_t x = c % W, y = c / W;
  switch (d) {
    case 0: return (ghost ? y - 1 : (y == 0 ? H - 1 : y - 1)) * W + x;
    case 1: return y * W + (x + 1 == W ? 0 : x + 1);
    case 2: return (ghost ? y + 1 : (y + 1 == H ? 0 : y + 1)) * W + x;
    default: return y * W + (x == 0 ? W - 1 : x - 1);
  }
}
__device__ __forceinline__ uint32_t wt_nbr(const dsr_wator_args& a, uint32_t c, uint32_t d) {
  return wt_nbr(a.W, a.H, c, d, a.ghost);
}
__device__ __forceinline__ bool wt_local(const dsr_wator_args& a, uint32_t c) {
  const uint32_t y = c / a.W;
  return !a.ghost || (y >= 1 && y <= a.H);
}
// global cell id (the RNG key index): local row y of the shard is global row y0 + y - 1
__device__ __forceinline__ uint32_t wt_gid(const dsr_wator_args& a, uint32_t c) {
  if (!a.ghost) return c;
  const uint32_t y = c / a.W, x = c % a.W;
  return ((a.y0 + y + a.Hg - 1) % a.Hg) * a.W + x;
}
// a ghost cell's agent: a handle whose type bits say Fish / Shark, never dereferenced
__device__ __forceinline__ uint64_t wt_ghost_agent(const DevHeap& h, uint32_t kind) {
  return kind ? make_handle(kind - 1, h.types[kind - 1].cap, 0, 0) : 0ull;
}
struct WtMig { uint32_t kind, egg, energy; };
__device__ __forceinline__ uint32_t wt_step(const dsr_wator_args& a) { return a.step_dev ? __ldg(a.step_dev) : a.step; }
__device__ __forceinline__ uint8_t* wt_halo(const dsr_wator_args& a, uint32_t off, uint32_t side) {
  return a.halo + off + side * a.W;
}
__device__ __forceinline__ WtMig* wt_mig(const dsr_wator_args& a, uint32_t off, uint32_t side) {
  return reinterpret_cast<WtMig*>(a.halo + off) + side * a.W;
}
__device__ __forceinline__ uint64_t* wt_agent(const DevHeap& h, const dsr_wator_args& a, uint32_t c) {
  return field_ptr<uint64_t>(h, a.cells[c], 1);
}
__device__ __forceinline__ uint8_t* wt_req(const DevHeap& h, const dsr_wator_args& a, uint32_t c, uint32_t k) {
  return field_ptr<uint8_t>(h, a.cells[c], 2 + k);
}
__device__ __forceinline__ uint32_t wt_pick(const uint32_t* list, uint32_t n, uint64_t key) {
  return list[(uint32_t)((key >> 32) % n)];
}

__device__ __forceinline__ uint64_t new_fish(const DevHeap& h, uint32_t c, uint32_t egg) {
  const uint64_t nh = dsr_new(h, WT_FISH);
  if (nh) {
    *field_ptr<uint32_t>(h, nh, 0) = c;
    *field_ptr<uint32_t>(h, nh, 1) = c;
    *field_ptr<uint32_t>(h, nh, 2) = egg;
  }
  return nh;
}
__device__ __forceinline__ uint64_t new_shark(const DevHeap& h, uint32_t c, uint32_t egg, uint32_t energy) {
  const uint64_t nh = dsr_new(h, WT_SHARK);
  if (nh) {
    *field_ptr<uint32_t>(h, nh, 0) = c;
    *field_ptr<uint32_t>(h, nh, 1) = c;
    *field_ptr<uint32_t>(h, nh, 2) = egg;
    *field_ptr<uint32_t>(h, nh, 3) = energy;
  }
  return nh;
}

// ---- parallel_new<Cell>(W*H): constructor i gets id i
__global__ void __launch_bounds__(256) k_wt_new_cells(DevHeap h, uint64_t n, dsr_wator_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    const uint64_t nh = dsr_new_bulk(h, WT_CELL, i < n);
    if (nh) {
      *field_ptr<uint32_t>(h, nh, 0) = (uint32_t)i;
      *field_ptr<uint64_t>(h, nh, 1) = 0;
      for (uint32_t k = 0; k < 5; ++k) *field_ptr<uint8_t>(h, nh, 2 + k) = 0;
    }
    if (i < n) a.cells[i] = nh;
  }
}
__global__ void __launch_bounds__(256) k_wt_init_agents(DevHeap h, uint64_t n, dsr_wator_args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // uniform trip count
    const uint64_t i = base + threadIdx.x;
    const uint32_t c = (uint32_t)i;
    uint8_t k = i < n ? a.kind0[c] : 0;
    if (k && !wt_local(a, c)) {                   // ghost row: the neighbour shard's agent kind
      *wt_agent(h, a, c) = wt_ghost_agent(h, k);
      k = 0;
    }
    const uint32_t T = k == 2 ? WT_SHARK : WT_FISH;
    const uint64_t nh = dsr_new_bulk(h, T, k != 0);
    if (nh) {
      *field_ptr<uint32_t>(h, nh, 0) = c;
      *field_ptr<uint32_t>(h, nh, 1) = c;
      *field_ptr<uint32_t>(h, nh, 2) = a.egg0[c];
      if (T == WT_SHARK) *field_ptr<uint32_t>(h, nh, 3) = a.energy0[c];
    }
    if (k) *wt_agent(h, a, c) = nh;
  }
}

struct WtCellPrepare {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args&, Acc&) {
#pragma unroll
    for (uint32_t k = 0; k < 5; ++k) *field_ptr<uint8_t>(h, T, 2 + k, b, s) = 0;
  }
};

template <int PHASE>
struct WtCellDecide {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    if (*field_ptr<uint8_t>(h, T, 6, b, s)) return;               // own agent stays
    uint32_t D[4], nd = 0;
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d)
      if (*field_ptr<uint8_t>(h, T, 2 + d, b, s)) D[nd++] = d;
    if (!nd) return;
    const uint32_t id = *field_ptr<uint32_t>(h, T, 0, b, s);
    if (!wt_local(a, id)) return;                                   // ghost cell: its owner decides
    const uint32_t d = wt_pick(D, nd, rng_key(a.seed, wt_step(a), PHASE, wt_gid(a, id)));
    const uint32_t nb = wt_nbr(a, id, d);
    if (!wt_local(a, nb)) {                                         // a neighbour shard's agent: grant it
      wt_halo(a, DSR_WT_HALO_GRANT_OUT(a.W), nb == id - a.W ? 0 : 1)[nb % a.W] = 1;
      return;
    }
    const uint64_t ag = *wt_agent(h, a, nb);
    *field_ptr<uint32_t>(h, ag, 1) = id;                            // Fish/Shark.target (field 1 of both)
  }
};

// The two Cell methods in quad form (k_doall_quad, reading C31):
// a lane owns 4 consecutive cells of a block; each u8 request column is one
// 32-bit word per quad (a warp's request is 128 B = 4 sectors instead of 32 B
// byte loads), stores only to the visited slots.
struct WtCellPrepareQ {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run4(const DevHeap& h, uint32_t T, uint32_t b, uint32_t q, uint32_t m4,
                                              const Args&, Acc&) {
    uint8_t* base = h.data + (size_t)b * h.block_bytes + 4u * q;
#pragma unroll
    for (uint32_t k = 0; k < 5; ++k) {
      uint8_t* col = base + h.types[T].col_off[2 + k];
      if (m4 == 0xFu) {
        *reinterpret_cast<uint32_t*>(col) = 0u;                 // columns are 16-B aligned (R-LAYOUT)
      } else {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j)
          if ((m4 >> j) & 1u) col[j] = 0;
      }
    }
  }
};
template <int PHASE>
struct WtCellDecideQ {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run4(const DevHeap& h, uint32_t T, uint32_t b, uint32_t q, uint32_t m4,
                                              const Args& a, Acc& acc) {
    const uint8_t* base = h.data + (size_t)b * h.block_bytes + 4u * q;
    uint32_t r[5];
#pragma unroll
    for (uint32_t k = 0; k < 5; ++k) r[k] = __ldg(reinterpret_cast<const uint32_t*>(base + h.types[T].col_off[2 + k]));
    // slots with a request and no "own agent stays" (req[4]) among the visited ones
    uint32_t todo = 0;
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
      const uint32_t any = ((r[0] | r[1] | r[2] | r[3]) >> (8 * j)) & 0xFFu;
      if (((m4 >> j) & 1u) && any && !((r[4] >> (8 * j)) & 0xFFu)) todo |= 1u << j;
    }
    while (todo) {
      const uint32_t j = __ffs(todo) - 1;
      todo &= todo - 1;
      uint32_t D[4], nd = 0;
#pragma unroll
      for (uint32_t d = 0; d < 4; ++d)
        if ((r[d] >> (8 * j)) & 0xFFu) D[nd++] = d;
      const uint32_t id = *reinterpret_cast<const uint32_t*>(base + h.types[T].col_off[0] + 12u * q + 4u * j);
      if (!wt_local(a, id)) continue;                                 // ghost cell: its owner decides
      const uint32_t d = wt_pick(D, nd, rng_key(a.seed, wt_step(a), PHASE, wt_gid(a, id)));
      const uint32_t nb = wt_nbr(a, id, d);
      if (!wt_local(a, nb)) {                                         // a neighbour shard's agent: grant it
        wt_halo(a, DSR_WT_HALO_GRANT_OUT(a.W), nb == id - a.W ? 0 : 1)[nb % a.W] = 1;
        continue;
      }
      const uint64_t ag = *wt_agent(h, a, nb);
      *field_ptr<uint32_t>(h, ag, 1) = id;                            // Fish/Shark.target (field 1 of both)
    }
  }
};

struct WtFishPrepare {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    *field_ptr<uint32_t>(h, T, 2, b, s) += 1;
    *field_ptr<uint32_t>(h, T, 1, b, s) = c;
    uint32_t fr[4], nf = 0;
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d)
      if (*wt_agent(h, a, wt_nbr(a, c, d)) == 0) fr[nf++] = d;
    if (nf) {
      const uint32_t d = wt_pick(fr, nf, rng_key(a.seed, wt_step(a), PH_FISH_REQ, wt_gid(a, c)));
      *wt_req(h, a, wt_nbr(a, c, d), d ^ 2) = 1;
    } else {
      *wt_req(h, a, c, 4) = 1;
    }
  }
};

struct WtFishUpdate {   // allocates Fish (snapshot pass)
  typedef dsr_wator_args Args;
  typedef Counters4 Acc;
  static __device__ __forceinline__ void flush(Acc& acc, const Args& a) { flush_counters4(acc, a.counters); }
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc& acc) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    const uint32_t t = *field_ptr<uint32_t>(h, T, 1, b, s);
    if (t == c) return;
    const bool away = !wt_local(a, t);                              // moves to a neighbour shard
    *wt_agent(h, a, c) = 0;
    if (!away) *wt_agent(h, a, t) = make_handle(T, h.types[T].cap, b, s);
    *field_ptr<uint32_t>(h, T, 0, b, s) = t;
    uint32_t* egg = field_ptr<uint32_t>(h, T, 2, b, s);
    if (*egg >= a.FB) {
      *egg = 0;
      *wt_agent(h, a, c) = new_fish(h, c, 0);
      acc.c[0] += 1;
    }
    if (away) {                                                     // migrate: the owner re-creates it
      wt_mig(a, DSR_WT_HALO_MIG_OUT(a.W), t < a.W ? 0 : 1)[t % a.W] = WtMig{1u, *egg, 0u};
      dsr_destroy(h, make_handle(T, h.types[T].cap, b, s));
    }
  }
};

struct WtSharkPrepare {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    *field_ptr<uint32_t>(h, T, 2, b, s) += 1;
    uint32_t* en = field_ptr<uint32_t>(h, T, 3, b, s);
    *en -= 1;
    *field_ptr<uint32_t>(h, T, 1, b, s) = c;
    if (*en == 0) return;                                           // starves in Shark.update
    uint32_t fd[4], nfd = 0, fr[4], nfr = 0;
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d) {
      const uint64_t ag = *wt_agent(h, a, wt_nbr(a, c, d));
      if (ag == 0) fr[nfr++] = d;
      else if (h_is(ag, WT_FISH)) fd[nfd++] = d;
    }
    const uint64_t key = rng_key(a.seed, wt_step(a), PH_SHARK_REQ, wt_gid(a, c));
    if (nfd) {
      const uint32_t d = wt_pick(fd, nfd, key);
      *wt_req(h, a, wt_nbr(a, c, d), d ^ 2) = 1;
    } else if (nfr) {
      const uint32_t d = wt_pick(fr, nfr, key);
      *wt_req(h, a, wt_nbr(a, c, d), d ^ 2) = 1;
    } else {
      *wt_req(h, a, c, 4) = 1;
    }
  }
};

struct WtSharkUpdate {  // allocates Shark (snapshot pass); destroys Fish and itself
  typedef dsr_wator_args Args;
  typedef Counters4 Acc;
  static __device__ __forceinline__ void flush(Acc& acc, const Args& a) { flush_counters4(acc, a.counters); }
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc& acc) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    const uint64_t self = make_handle(T, h.types[T].cap, b, s);
    uint32_t* en = field_ptr<uint32_t>(h, T, 3, b, s);
    if (*en == 0) {
      *wt_agent(h, a, c) = 0;
      dsr_destroy(h, self);                                         // self-delete
      acc.c[3] += 1;
      return;
    }
    const uint32_t t = *field_ptr<uint32_t>(h, T, 1, b, s);
    if (t == c) return;
    const bool away = !wt_local(a, t);                              // moves to a neighbour shard (which
    uint64_t* at = wt_agent(h, a, t);                               // resolves the prey on arrival)
    if (!away) {
      const uint64_t prey = *at;
      if (prey && h_is(prey, WT_FISH)) {
        dsr_destroy(h, prey);                                       // another type
        *en = a.SS;
        acc.c[2] += 1;
      }
    }
    *wt_agent(h, a, c) = 0;
    if (!away) *at = self;
    *field_ptr<uint32_t>(h, T, 0, b, s) = t;
    uint32_t* egg = field_ptr<uint32_t>(h, T, 2, b, s);
    if (*egg >= a.SB) {
      *egg = 0;
      *wt_agent(h, a, c) = new_shark(h, c, 0, a.SS);
      acc.c[1] += 1;
    }
    if (away) {
      wt_mig(a, DSR_WT_HALO_MIG_OUT(a.W), t < a.W ? 0 : 1)[t % a.W] = WtMig{2u, *egg, *en};
      dsr_destroy(h, self);
    }
  }
};

// ---- row sharding: the boundary stages of a half step
__global__ void k_wt_req_pack(DevHeap h, uint64_t n, dsr_wator_args a) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.W; x += gridDim.x * blockDim.x) {
    wt_halo(a, DSR_WT_HALO_REQ_OUT(a.W), 0)[x] = *wt_req(h, a, x, 2);                    // ghost row 0: from my row 1
    wt_halo(a, DSR_WT_HALO_REQ_OUT(a.W), 1)[x] = *wt_req(h, a, (a.H + 1) * a.W + x, 0);  // ghost row H+1
    for (uint32_t sd = 0; sd < 2; ++sd) {
      wt_halo(a, DSR_WT_HALO_GRANT_OUT(a.W), sd)[x] = 0;
      wt_mig(a, DSR_WT_HALO_MIG_OUT(a.W), sd)[x] = WtMig{0u, 0u, 0u};
    }
  }
}
__global__ void k_wt_req_apply(DevHeap h, uint64_t n, dsr_wator_args a) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.W; x += gridDim.x * blockDim.x) {
    if (wt_halo(a, DSR_WT_HALO_REQ_IN(a.W), 0)[x]) *wt_req(h, a, a.W + x, 0) = 1;        // from the agent above
    if (wt_halo(a, DSR_WT_HALO_REQ_IN(a.W), 1)[x]) *wt_req(h, a, a.H * a.W + x, 2) = 1;  // from the agent below
  }
}
__global__ void k_wt_grant_apply(DevHeap h, uint64_t n, dsr_wator_args a) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.W; x += gridDim.x * blockDim.x) {
    if (wt_halo(a, DSR_WT_HALO_GRANT_IN(a.W), 0)[x])
      *field_ptr<uint32_t>(h, *wt_agent(h, a, a.W + x), 1) = x;                           // -> ghost row 0
    if (wt_halo(a, DSR_WT_HALO_GRANT_IN(a.W), 1)[x])
      *field_ptr<uint32_t>(h, *wt_agent(h, a, a.H * a.W + x), 1) = (a.H + 1) * a.W + x;  // -> ghost row H+1
  }
}
__global__ void __launch_bounds__(256) k_wt_mig_apply(DevHeap h, uint64_t n, dsr_wator_args a) {
  const uint32_t n2 = 2 * a.W, stride = gridDim.x * blockDim.x;
  unsigned long long eaten = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n2; base += stride) {   // uniform trip count
    const uint32_t i = base + threadIdx.x;
    WtMig m{0u, 0u, 0u};
    uint32_t c = 0;
    if (i < n2) {
      const uint32_t sd = i / a.W, x = i % a.W;
      m = wt_mig(a, DSR_WT_HALO_MIG_IN(a.W), sd)[x];
      c = (sd ? a.H : 1u) * a.W + x;                               // arrival cell on my boundary row
    }
    if (m.kind == 2) {
      const uint64_t prey = *wt_agent(h, a, c);
      if (prey && h_is(prey, WT_FISH)) {                            // the shark eats on arrival
        dsr_destroy(h, prey);
        m.energy = a.SS;
        ++eaten;
      }
    }
    const uint32_t T = m.kind == 2 ? WT_SHARK : WT_FISH;
    const uint64_t nh = dsr_new_bulk(h, T, m.kind != 0);
    if (nh) {
      *field_ptr<uint32_t>(h, nh, 0) = c;
      *field_ptr<uint32_t>(h, nh, 1) = c;
      *field_ptr<uint32_t>(h, nh, 2) = m.egg;
      if (T == WT_SHARK) *field_ptr<uint32_t>(h, nh, 3) = m.energy;
    }
    if (m.kind) *wt_agent(h, a, c) = nh;
  }
  if (eaten) atomicAdd(&a.counters[2], eaten);
}
__device__ __forceinline__ uint8_t wt_kind(uint64_t ag) { return ag == 0 ? 0 : (h_is(ag, WT_FISH) ? 1 : 2); }
__global__ void k_wt_occ_pack(DevHeap h, uint64_t n, dsr_wator_args a) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.W; x += gridDim.x * blockDim.x) {
    wt_halo(a, DSR_WT_HALO_OCC_OUT(a.W), 0)[x] = wt_kind(*wt_agent(h, a, a.W + x));
    wt_halo(a, DSR_WT_HALO_OCC_OUT(a.W), 1)[x] = wt_kind(*wt_agent(h, a, a.H * a.W + x));
  }
}
__global__ void k_wt_occ_apply(DevHeap h, uint64_t n, dsr_wator_args a) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.W; x += gridDim.x * blockDim.x) {
    *wt_agent(h, a, x) = wt_ghost_agent(h, wt_halo(a, DSR_WT_HALO_OCC_IN(a.W), 0)[x]);
    *wt_agent(h, a, (a.H + 1) * a.W + x) = wt_ghost_agent(h, wt_halo(a, DSR_WT_HALO_OCC_IN(a.W), 1)[x]);
  }
}

struct WtDump {
  typedef dsr_wator_args Args;
  DSR_NO_ACC
  static __device__ __forceinline__ void run(const DevHeap& h, uint32_t T, uint32_t b, uint32_t s, const Args& a, Acc&) {
    const uint32_t c = *field_ptr<uint32_t>(h, T, 0, b, s);
    a.out_kind[c] = T == WT_FISH ? 1u : 2u;
    a.out_egg[c] = *field_ptr<uint32_t>(h, T, 2, b, s);
    a.out_energy[c] = T == WT_SHARK ? *field_ptr<uint32_t>(h, T, 3, b, s) : 0u;
  }
};

bool wt_method_info(uint32_t id, MethodInfo* mi) {
  switch (id) {
    case DSR_M_WT_CELL_PREPARE: case DSR_M_WT_FISH_PREPARE: case DSR_M_WT_CELL_DECIDE_FISH:
    case DSR_M_WT_SHARK_PREPARE: case DSR_M_WT_CELL_DECIDE_SHARK: case DSR_M_WT_DUMP:
      *mi = {0, sizeof(dsr_wator_args)}; return true;
    case DSR_M_WT_FISH_UPDATE: case DSR_M_WT_SHARK_UPDATE:
      *mi = {1, sizeof(dsr_wator_args)}; return true;
  }
  return false;
}

bool wt_method_launch(uint32_t id, const LaunchCtx& c, uint32_t T, int snapshot, const void* args) {
  switch (id) {
    case DSR_M_WT_CELL_PREPARE:
      if (c.h.flags & DSR_F_SCALAR_DOALL) launch_doall<WtCellPrepare>(c, T, snapshot, args);
      else launch_doall_quad<WtCellPrepareQ>(c, T, snapshot, args);
      return true;
    case DSR_M_WT_FISH_PREPARE: launch_doall<WtFishPrepare>(c, T, snapshot, args); return true;
    case DSR_M_WT_CELL_DECIDE_FISH:
      if (c.h.flags & DSR_F_SCALAR_DOALL) launch_doall<WtCellDecide<PH_FISH_DEC>>(c, T, snapshot, args);
      else launch_doall_quad<WtCellDecideQ<PH_FISH_DEC>>(c, T, snapshot, args);
      return true;
    case DSR_M_WT_FISH_UPDATE: launch_doall<WtFishUpdate>(c, T, snapshot, args); return true;
    case DSR_M_WT_SHARK_PREPARE: launch_doall<WtSharkPrepare>(c, T, snapshot, args); return true;
    case DSR_M_WT_CELL_DECIDE_SHARK:
      if (c.h.flags & DSR_F_SCALAR_DOALL) launch_doall<WtCellDecide<PH_SHARK_DEC>>(c, T, snapshot, args);
      else launch_doall_quad<WtCellDecideQ<PH_SHARK_DEC>>(c, T, snapshot, args);
      return true;
    case DSR_M_WT_SHARK_UPDATE: launch_doall<WtSharkUpdate>(c, T, snapshot, args); return true;
    case DSR_M_WT_DUMP: launch_doall<WtDump>(c, T, snapshot, args); return true;
  }
  return false;
}

bool wt_kernel_launch(uint32_t id, const LaunchCtx& c, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id < DSR_K_WT_INIT_AGENTS || id > DSR_K_WT_HALO_OCC_APPLY) return false;
  if (bytes != sizeof(dsr_wator_args) || c.h.ntypes < 3) { *ok = 0; return true; }
  const dsr_wator_args a = *(const dsr_wator_args*)args;
  if (id == DSR_K_WT_INIT_AGENTS) {
    if ((uint64_t)a.W * (a.H + (a.ghost ? 2 : 0)) != n) { *ok = 0; return true; }
    k_wt_init_agents<<<grid_for(c, n, k_wt_init_agents), 256, 0, c.st>>>(c.h, n, a);
    count_launch();
    return true;
  }
  if (!a.ghost || !a.halo || n != a.W || a.H == 0 || a.Hg == 0) { *ok = 0; return true; }
  switch (id) {
    case DSR_K_WT_HALO_REQ_PACK: k_wt_req_pack<<<grid_for(c, n, k_wt_req_pack), 256, 0, c.st>>>(c.h, n, a); break;
    case DSR_K_WT_HALO_REQ_APPLY: k_wt_req_apply<<<grid_for(c, n, k_wt_req_apply), 256, 0, c.st>>>(c.h, n, a); break;
    case DSR_K_WT_HALO_GRANT_APPLY:
      k_wt_grant_apply<<<grid_for(c, n, k_wt_grant_apply), 256, 0, c.st>>>(c.h, n, a); break;
    case DSR_K_WT_HALO_MIG_APPLY: k_wt_mig_apply<<<grid_for(c, 2 * n, k_wt_mig_apply), 256, 0, c.st>>>(c.h, n, a); break;
    case DSR_K_WT_HALO_OCC_PACK: k_wt_occ_pack<<<grid_for(c, n, k_wt_occ_pack), 256, 0, c.st>>>(c.h, n, a); break;
    default: k_wt_occ_apply<<<grid_for(c, n, k_wt_occ_apply), 256, 0, c.st>>>(c.h, n, a); break;
  }
  count_launch();
  return true;
}

bool wt_ctor_launch(uint32_t id, const LaunchCtx& c, uint32_t T, uint64_t n, const void* args, size_t bytes, int* ok) {
  *ok = 1;
  if (id != DSR_C_WT_CELL) return false;
  if (bytes != sizeof(dsr_wator_args) || T != WT_CELL || c.h.ntypes < 3) { *ok = 0; return true; }
  const dsr_wator_args a = *(const dsr_wator_args*)args;
  if ((uint64_t)a.W * (a.H + (a.ghost ? 2 : 0)) != n) { *ok = 0; return true; }
  k_wt_new_cells<<<grid_for(c, n, k_wt_new_cells), 256, 0, c.st>>>(c.h, n, a);
  count_launch();
  return true;
}

}  // namespace dsr
