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
static void bitmap_shape(uint64_t n, uint32_t* nlevels, uint64_t* words, uint64_t* total) {
  uint32_t l = 0;
  uint64_t tot = 0, size = n;
  for (;;) {
    uint64_t w = (size + 63) / 64;
    if (w == 0) w = 1;
    words[l] = w;
    tot += w;
    l++;
    if (size <= 64) break;
    size = w;
  }
  *nlevels = l;
  *total = tot;
}

/* Byte size of every region for a given M, in the order of DESIGN.md "HBM
 * layout": control page, data, alloc_bm, iter_bm, type, R, bitmaps. */
/* control page (4 KiB) + per-warp block-hint table of H slots x 8 types x
 * u32, H = pow2floor(heap_bytes / 64 KiB) clamped to [64, 16384] (R-LAYOUT) */
static uint64_t ctrl_bytes(uint64_t heap_bytes) {
  uint64_t h = 64;
  while (h * 2 <= (heap_bytes >> 16) && h < 16384) h *= 2;
  return 4096 + h * 8 * 4;
}

static uint64_t layout_for_M(or_layout_t* L, uint64_t M, uint64_t heap_bytes) {
  uint64_t off = ctrl_bytes(heap_bytes);
  L->M = M;
  L->off_data = off;       off = align_up(off + M * (uint64_t)L->block_bytes, 256);
  L->off_alloc_bm = off;   off = align_up(off + M * 8, 256);
  L->off_iter_bm = off;    off = align_up(off + M * 8, 256);
  L->off_type = off;       off = align_up(off + M * 1, 256);
  L->off_R = off;          off = align_up(off + M * 4, 256);
  uint64_t total_words = 0;
  bitmap_shape(M ? M : 1, &L->nlevels, L->level_words, &total_words);
  L->bitmap_words = align_up(total_words, 32);  /* each bitmap 256-B aligned */
  L->off_bitmaps = off;
  off += (1 + 2 * (uint64_t)L->ntypes) * L->bitmap_words * 8;
  L->total_bytes = off;
  return off;
}

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
  /* block capacity N_T = floor(64 * size(T_s) / size(T)) */
  uint64_t data_max = 0;
  for (uint32_t t = 0; t < ntypes; t++) {
    uint64_t cap = 64 * smin / size[t];
    if (cap < 1) return 2;                       /* "more than 64 times bigger" P:313 */
    L->cap[t] = (uint32_t)cap;
    /* SOA columns packed back to back, each 16-byte aligned (R-LAYOUT: a
     * 128-bit vector load per column segment; the block is 128-aligned) */
    uint64_t off = 0, end = 0;
    for (uint32_t f = 0; f < L->nfields[t]; f++) {
      uint64_t colb = cap * L->fsize[t][f];
      off = align_up(end, 16);
      L->col_off[t][f] = (uint32_t)off;
      end = off + colb;
    }
    if (end > data_max) data_max = end;
  }
  L->block_bytes = (uint32_t)align_up(data_max, 128);
  /* M = the largest block count whose regions fit in heap_bytes (monotone). */
  uint64_t lo = 0, hi = heap_bytes / L->block_bytes + 1;
  if (hi > 0xFFFFFFFFULL) hi = 0xFFFFFFFFULL;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo + 1) / 2;
    if (layout_for_M(L, mid, heap_bytes) <= heap_bytes) lo = mid; else hi = mid - 1;
  }
  if (lo == 0) return 3;
  layout_for_M(L, lo, heap_bytes);
  return 0;
}
