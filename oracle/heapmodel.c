/*
 * oracle/heapmodel.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Sequential (one-thread) execution of the paper's allocator:
 *   Alg. 1 allocate<T>
 *   Alg. 2 deallocate<T>      P:404-426 (+ reading R-FIRSTEMPTY / C17)
 *   Alg. 6 Block::reserve     P:659-685 (padding generalisation R-PAD / C5)
 *   Alg. 7 Block::deallocate
 *   Alg. 8 initialize_block
 *   Alg. 9 invalidate
 *   block bitmaps             P:346-353 (free all 1, allocated/active all 0)
 *   object pointer            Fig. 5; Listing 2 P:1252-1256 (C6/C7)
 * Used for single-thread replay: the CUDA heap run by one thread with
 * rotation off must produce the same words, types and handles.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

struct or_heap {
  or_layout_t L;
  uint64_t* alloc_bm;      /* object allocation bitmap per block */
  uint8_t* type;           /* type identifier per block, 0 = never initialised */
  or_bitmap_t* freebm;     /* free block bitmap */
  or_bitmap_t* allocated[OR_MAXT];
  or_bitmap_t* active[OR_MAXT];
  int error;
  or_hook_fn hook;         /* scripted interleavings (tests) */
  void* hook_ctx;
  uint32_t hook_armed;     /* bit p: call the hook at point p once */
  uint64_t counters[4];
};

void or_heap_set_hook(or_heap_t* h, or_hook_fn fn, void* ctx, uint32_t point) {
  h->hook = fn;
  h->hook_ctx = ctx;
  h->hook_armed |= 1u << point;
}
uint64_t or_heap_counter(const or_heap_t* h, uint32_t k) { return k < 4 ? h->counters[k] : 0; }
static void fire(or_heap_t* h, uint32_t point, uint64_t bid) {
  if (h->hook && (h->hook_armed & (1u << point))) {
    h->hook_armed &= ~(1u << point);
    h->hook(h->hook_ctx, point, bid);
  }
}

/* type ids are 1-based in handles and type[] (reading R-TYPEID / C18) */
static uint64_t pad_mask(uint32_t cap) { return cap == 64 ? 0ULL : ~((1ULL << cap) - 1); }

/* Fig. 5 / Listing 2: slot bits 0-5 (mask 0x3F), block bits 6-49
 * (mask 0x3FFFFFFFFFFC0), capacity bits 50-55 ((p & 0xFC000000000000) >> 50),
 * type id bits 56-63.  Capacity is stored as N_T - 1 (reading R-CAP / C6) and
 * bits 6-49 hold the block index, not an address (reading R-BID / C7). */
uint64_t or_handle_encode(uint32_t type, uint32_t cap, uint64_t bid, uint32_t slot) {
  return ((uint64_t)type << 56) | ((uint64_t)(cap - 1) << 50) | (bid << 6) | (uint64_t)slot;
}
void or_handle_decode(uint64_t h, uint32_t* type, uint32_t* cap, uint64_t* bid, uint32_t* slot) {
  *slot = (uint32_t)(h & 0x3F);
  *bid = (h & 0x3FFFFFFFFFFC0ULL) >> 6;
  *cap = (uint32_t)((h & 0xFC000000000000ULL) >> 50) + 1;
  *type = (uint32_t)(h >> 56);
}

or_heap_t* or_heap_new(uint32_t ntypes, const uint32_t* nfields, const uint32_t* fsizes_flat, uint64_t M) {
  or_heap_t* h = (or_heap_t*)calloc(1, sizeof(or_heap_t));
  /* capacities from the layout; the block count is the caller's */
  if (M == 0 || or_layout(ntypes, nfields, fsizes_flat, 1ULL << 40, &h->L) != 0) { free(h); return NULL; }
  h->L.M = M;
  h->alloc_bm = (uint64_t*)malloc(M * sizeof(uint64_t));
  /* uninitialised blocks behave like invalidated ones: all bits 1 */
  for (uint64_t b = 0; b < M; b++) h->alloc_bm[b] = ~0ULL;
  h->type = (uint8_t*)calloc(M, 1);
  h->freebm = or_bm_new(M, 64, 1);                     /* "Initially, every bit is 1" P:350 */
  for (uint32_t t = 0; t < ntypes; t++) {
    h->allocated[t] = or_bm_new(M, 64, 0);             /* "Initially, every bit is 0" P:351 */
    h->active[t] = or_bm_new(M, 64, 0);
  }
  return h;
}

void or_heap_free(or_heap_t* h) {
  if (!h) return;
  free(h->alloc_bm);
  free(h->type);
  or_bm_free(h->freebm);
  for (uint32_t t = 0; t < h->L.ntypes; t++) { or_bm_free(h->allocated[t]); or_bm_free(h->active[t]); }
  free(h);
}

/* Alg. 8: type <- T; threadfence; bitmap <- 0 (padding bits 1, App. A.1) */
static void initialize_block(or_heap_t* h, uint32_t T, uint64_t bid) {
  h->type[bid] = (uint8_t)(T + 1);
  h->alloc_bm[bid] = pad_mask(h->L.cap[T]);
}

/* Alg. 6: pos <- ffs(~bitmap); before <- atomicOr(mask); FULL iff the
 * reservation filled the last free bit ((before | mask) == ~0, R-PAD). */
static int reserve(or_heap_t* h, uint64_t bid, uint32_t* slot, int* full) {
  uint64_t bm = h->alloc_bm[bid];
  if (~bm == 0) return 0;                    /* pos = NONE -> FAIL */
  uint32_t pos = (uint32_t)__builtin_ctzll(~bm);
  uint64_t mask = 1ULL << pos;
  uint64_t before = bm;
  h->alloc_bm[bid] = before | mask;
  *slot = pos;
  *full = ((before | mask) == ~0ULL);
  return 1;
}

/* Alg. 9 with padding: success iff all non-padding bits were 0 before. */
static int invalidate(or_heap_t* h, uint64_t bid) {
  for (;;) {
    uint64_t before = h->alloc_bm[bid];
    h->alloc_bm[bid] = ~0ULL;                             /* atomicOr(0xFF..F) */
    if (before == ~0ULL) return 0;
    uint32_t t = h->type[bid] - 1u;
    if (before == pad_mask(h->L.cap[t])) return 1;
    h->counters[1]++;
    fire(h, OR_HOOK_INVALIDATED, bid);
    uint64_t before_rb = h->alloc_bm[bid];
    h->alloc_bm[bid] = before_rb & before;                /* rollback */
    if (before_rb != ~0ULL) {                             /* deferred deactivation (l.10) */
      or_bm_clear(h->active[t], 0, bid);
      h->counters[3]++;
    }
    if ((before_rb & before) == pad_mask(h->L.cap[t])) { h->counters[2]++; continue; }   /* empty again */
    return 0;
  }
}

/* Alg. 7 + Alg. 2 (with FIRST and EMPTY at once: set active, then try to
 * invalidate -- reading R-FIRSTEMPTY / C17). */
static void dealloc_block(or_heap_t* h, uint32_t T, uint64_t bid, uint64_t mask) {
  uint64_t before = h->alloc_bm[bid];
  if ((before & mask) != mask) { h->error = 2; return; }    /* assert(success) P:1000 */
  h->alloc_bm[bid] = before & ~mask;
  int first = (before == ~0ULL);                             /* popc(before) = 64 */
  int empty = ((before & ~mask) == pad_mask(h->L.cap[T]));   /* popc(before) = 1 */
  if (first) or_bm_set(h->active[T], 0, bid);
  if (empty) {
    fire(h, OR_HOOK_EMPTIED, bid);
    if (invalidate(h, bid)) {
      uint32_t t = h->type[bid] - 1u;
      or_bm_clear(h->active[t], 0, bid);
      or_bm_clear(h->allocated[t], 0, bid);
      or_bm_set(h->freebm, 0, bid);
    }
  }
}

/* Alg. 1 (r attempts collapse to one in sequential execution: a consistent
 * bitmap never FAILs spuriously). */
uint64_t or_heap_alloc(or_heap_t* h, uint32_t T) {
  if (T >= h->L.ntypes) return 0;
  for (;;) {
    int64_t bid = or_bm_try_find_set(h->active[T], 0);
    if (bid < 0) {                                         /* slow path */
      bid = or_bm_clear_any(h->freebm);
      if (bid < 0) return 0;                               /* OOM (reading R-OOM / C14) */
      initialize_block(h, T, (uint64_t)bid);
      or_bm_set(h->allocated[T], 0, (uint64_t)bid);
      or_bm_set(h->active[T], 0, (uint64_t)bid);
    }
    fire(h, OR_HOOK_FOUND, (uint64_t)bid);
    uint32_t slot;
    int full;
    if (reserve(h, (uint64_t)bid, &slot, &full)) {
      uint32_t t = h->type[bid] - 1u;                      /* volatile read */
      if (full) or_bm_clear(h->active[t], 0, (uint64_t)bid);
      if (t == T) return or_handle_encode(T + 1, h->L.cap[T], (uint64_t)bid, slot);
      h->counters[0]++;
      dealloc_block(h, t, (uint64_t)bid, 1ULL << slot);    /* rollback (l.14) */
    }
  }
}

int or_heap_dealloc(or_heap_t* h, uint64_t handle) {
  uint32_t type, cap, slot;
  uint64_t bid;
  or_handle_decode(handle, &type, &cap, &bid, &slot);
  if (type < 1 || type > h->L.ntypes || bid >= h->L.M) return 1;
  dealloc_block(h, type - 1, bid, 1ULL << slot);
  return h->error;
}

uint64_t or_heap_M(const or_heap_t* h) { return h->L.M; }
uint64_t or_heap_alloc_bm(const or_heap_t* h, uint64_t bid) { return h->alloc_bm[bid]; }
uint32_t or_heap_type(const or_heap_t* h, uint64_t bid) { return h->type[bid]; }
or_bitmap_t* or_heap_bitmap(or_heap_t* h, uint32_t which, uint32_t t) {
  if (which == 0) return h->freebm;
  if (t >= h->L.ntypes) return NULL;
  return which == 1 ? h->allocated[t] : h->active[t];
}

/* live(T) = sum over allocated[T] blocks of used slots */
uint64_t or_heap_live(const or_heap_t* h, uint32_t t) {
  uint64_t n = 0;
  for (uint64_t b = 0; b < h->L.M; b++)
    if (or_bm_get(h->allocated[t], b))
      n += (uint64_t)__builtin_popcountll(h->alloc_bm[b] & ~pad_mask(h->L.cap[t]));
  return n;
}

/* fragmentation F: unused slots / total slots over allocated blocks;
 * 0 when no block is allocated (reading C36). */
double or_heap_fragmentation(const or_heap_t* h) {
  uint64_t unused = 0, total = 0;
  for (uint32_t t = 0; t < h->L.ntypes; t++)
    for (uint64_t b = 0; b < h->L.M; b++)
      if (or_bm_get(h->allocated[t], b)) {
        uint32_t used = (uint32_t)__builtin_popcountll(h->alloc_bm[b] & ~pad_mask(h->L.cap[t]));
        unused += h->L.cap[t] - used;
        total += h->L.cap[t];
      }
  return total ? (double)unused / (double)total : 0.0;
}

int or_heap_error(const or_heap_t* h) {
  int e = h->error | h->freebm->error;
  for (uint32_t t = 0; t < h->L.ntypes; t++) e |= h->allocated[t]->error | h->active[t]->error;
  return e;
}

/* ---- thread assignment, P:471-479 ----
 * id_O(tid) = tid % N_T; id_B(tid) = R[(tid + k n) / N_T], k < num_B(tid);
 * num_B(tid) = ceil((r N_T - tid) / n), clamped at 0 (reading R-ASSIGN / C9). */
uint64_t or_assign_num_blocks(uint64_t r, uint32_t NT, uint64_t n, uint64_t tid) {
  uint64_t tot = r * NT;
  if (tid >= tot) return 0;
  return (tot - tid + n - 1) / n;
}
uint64_t or_assign_block_pos(uint32_t NT, uint64_t n, uint64_t tid, uint64_t k) {
  return (tid + k * n) / NT;
}
/* slot of the k-th assignment: (tid + k n) % N_T, which is the paper's
 * id_O(tid) = tid % N_T whenever n = 0 (mod N_T). */
uint32_t or_assign_slot(uint32_t NT, uint64_t n, uint64_t tid, uint64_t k) {
  return (uint32_t)((tid + k * n) % NT);
}
