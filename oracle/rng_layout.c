/*
 * oracle/rng_layout.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Counter-based RNG (reading R-RNG, SURVEY c.5) and the heap layout
 * ("heap is divided into M blocks", P:305-313 block capacity,
 * P:228 128-byte clusters, readings R-LAYOUT / C20 in DESIGN.md).
 */
#include "oracle.h"
#include <string.h>

/* SplitMix64 output function applied to x (Steele/Lea/Flood; Vigna's
 * splitmix64.c next() with state x before the increment).  Reading R-RNG. */
uint64_t or_sm(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* key(seed, step, phase, idx) = sm(sm(sm(seed) ^ step) ^ (phase<<40 | idx)) */
uint64_t or_key(uint64_t seed, uint64_t step, uint64_t phase, uint64_t idx) {
  return or_sm(or_sm(or_sm(seed) ^ step) ^ ((phase << 40) | idx));
}

static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

/* Number of levels and words of a hierarchical bitmap of n bits with 64-bit
 * containers: "an array of size ceil(N/64) of 64-bit containers, and a nested
 * bitmap of size ceil(N/64) if N > 64". */
static void bitmap_shape(uint64_t n, uint32_t* nlevels, uint64_t* words) {
  uint32_t l = 0;
  uint64_t size = n;
  for (;;) {
    uint64_t w = (size + 63) / 64;
    if (w == 0) w = 1;
    words[l++] = w;
    if (size <= 64) break;
    size = w;
  }
  *nlevels = l;
}

/* Heap layout of `ntypes` types in heap_bytes (what the paper fixes, and the
 * DESIGN.md reading R-LAYOUT where it does not):
 *   N_T = floor(64 size(T_s) / size(T))
 *   the data segment of a block holds N_T objects of its type as SOA arrays,
 *   inherited fields first; R-LAYOUT: column f of T starts at the
 *   next 16-byte boundary after column f-1 (packed; 16 B = one vector load),
 *   a block's data segment is the largest type's, rounded up to 128 B (a
 *   cache line), "every block has the same byte size";
 *   M = the number of blocks a heap of heap_bytes can hold when every block
 *   also carries the state the paper gives it: the allocation and iteration
 *   bitmaps (8 B each), the type identifier (1 B), its entry of
 *   the do-all block-index array (4 B) and one bit in each of the
 *   1 + 2 ntypes block bitmaps free / allocated[T] / active[T]:
 *     M = floor(8 heap_bytes / (8 (block_bytes + 21) + 1 + 2 ntypes)).
 *   The nested levels of the block bitmaps and any fixed header are not
 *   counted, so an implementation's M is at most this bound (and close to it).
 *   Levels of an M-bit bitmap follow P:501. */
int or_layout(uint32_t ntypes, const uint32_t* nfields, const uint32_t* fsizes_flat,
              uint64_t heap_bytes, or_layout_t* L) {
  memset(L, 0, sizeof(*L));
  if (ntypes < 1 || ntypes > OR_MAXT) return 1;
  L->ntypes = ntypes;
  uint64_t size[OR_MAXT], smin = ~0ULL;
  uint32_t k = 0;
  for (uint32_t t = 0; t < ntypes; t++) {
    if (nfields[t] < 1 || nfields[t] > OR_MAXF) return 1;
    L->nfields[t] = nfields[t];
    size[t] = 0;
    for (uint32_t f = 0; f < nfields[t]; f++) {
      uint32_t s = fsizes_flat[k++];
      if (!(s == 1 || s == 2 || s == 4 || s == 8 || s == 16)) return 1;
      L->fsize[t][f] = s;
      size[t] += s;
    }
    if (size[t] < smin) smin = size[t];
  }
  uint64_t data_max = 0;
  for (uint32_t t = 0; t < ntypes; t++) {
    uint64_t cap = 64 * smin / size[t];
    if (cap < 1) return 2;                       /* "more than 64 times bigger" P:313 */
    L->cap[t] = (uint32_t)cap;
    uint64_t end = 0;
    for (uint32_t f = 0; f < L->nfields[t]; f++) {
      uint64_t off = align_up(end, 16);
      L->col_off[t][f] = (uint32_t)off;
      end = off + cap * L->fsize[t][f];
    }
    if (end > data_max) data_max = end;
  }
  L->block_bytes = (uint32_t)align_up(data_max, 128);
  L->M = 8 * heap_bytes / (8 * ((uint64_t)L->block_bytes + 21) + 1 + 2 * (uint64_t)ntypes);
  if (L->M == 0) return 3;
  bitmap_shape(L->M, &L->nlevels, L->level_words);
  return 0;
}
