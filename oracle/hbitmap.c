/*
 * oracle/hbitmap.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Sequential hierarchical bitmap with a container width W parameter
 * (W = 64 in DynaSOAr; W = 4 reproduces Fig. 7).
 *
 *   data structure  : P:500-505  (containers + nested bitmap if N > W)
 *   try_clear       : Alg. 3, P:534-559 (cascade clear when popc(prev) = 1)
 *   try_set         : "symmetric" to try_clear (Def. P:1126-1131 set-first)
 *   set / clear     : "retries until the bit was changed"; higher
 *                     levels always use the retrying versions
 *   try_find_set    : Alg. 4, P:561-591 (top-down; NoShift, i.e. plain ffs)
 *   clear()         : P:529, reading R-CLEARANY (retry while try_clear fails)
 *   indices         : Alg. 5, P:592-621 (uses the nested level to skip)
 *   consistency     : Definition
 * Sequential execution: a set / clear that finds its bit already in the
 * target state waits (pending) for the opposite op, as the paper's spinning
 * thread would; one never released is the paper's deadlock (illegal use,
 * P:1146) and makes or_bm_error report it.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

static uint64_t wmask(uint32_t W) { return W == 64 ? ~0ULL : ((1ULL << W) - 1); }

or_bitmap_t* or_bm_new(uint64_t n, uint32_t W, int all_set) {
  if (n < 1 || W < 2 || W > 64) return NULL;
  or_bitmap_t* b = (or_bitmap_t*)calloc(1, sizeof(or_bitmap_t));
  b->n = n;
  b->W = W;
  uint64_t size = n;
  uint32_t l = 0;
  for (;;) {
    b->size[l] = size;
    uint64_t words = (size + W - 1) / W;
    b->c[l] = (uint64_t*)calloc(words, sizeof(uint64_t));
    l++;
    if (size <= W) break;          /* nested bitmap only "if N > 64" */
    size = words;
  }
  b->nlevels = l;
  if (all_set) {
    /* every real bit 1; bits >= size stay 0 (reading R-PAD / C2) */
    for (uint32_t lv = 0; lv < b->nlevels; lv++)
      for (uint64_t i = 0; i < b->size[lv]; i++)
        b->c[lv][i / W] |= 1ULL << (i % W);
  }
  return b;
}

void or_bm_free(or_bitmap_t* b) {
  if (!b) return;
  for (uint32_t l = 0; l < b->nlevels; l++) free(b->c[l]);
  free(b);
}

static void trace(or_bitmap_t* b, uint32_t level, uint64_t pos, uint32_t is_set) {
  if (b->trace_on && b->ntrace < 64) {
    b->trace[b->ntrace][0] = level;
    b->trace[b->ntrace][1] = (uint32_t)pos;
    b->trace[b->ntrace][2] = is_set;
    b->ntrace++;
  }
}

/* the op waiting on (level, pos) for the opposite state, if any, completes now */
static void resolve_pending(or_bitmap_t* b, uint32_t level, uint64_t pos, uint32_t want_set) {
  for (uint32_t i = 0; i < b->npend; i++) {
    if (b->pend_lvl[i] == level && b->pend_pos[i] == pos && b->pend_set[i] == want_set) {
      b->npend--;
      b->pend_lvl[i] = b->pend_lvl[b->npend];
      b->pend_pos[i] = b->pend_pos[b->npend];
      b->pend_set[i] = b->pend_set[b->npend];
      if (want_set) or_bm_try_set(b, level, pos); else or_bm_try_clear(b, level, pos);
      return;
    }
  }
}
static void add_pending(or_bitmap_t* b, uint32_t level, uint64_t pos, uint32_t is_set) {
  if (b->npend == 16) { b->error = 1; return; }
  b->pend_lvl[b->npend] = level;
  b->pend_pos[b->npend] = pos;
  b->pend_set[b->npend] = is_set;
  b->npend++;
}

/* Alg. 3: prev <- atomicAnd(&container[cid], ~mask); success <- prev & mask;
 * if success and has_nested and popc(prev) = 1: nested.clear(cid). */
int or_bm_try_clear(or_bitmap_t* b, uint32_t level, uint64_t pos) {
  uint64_t cid = pos / b->W, mask = 1ULL << (pos % b->W);
  uint64_t prev = b->c[level][cid];
  b->c[level][cid] = prev & ~mask;
  int success = (prev & mask) != 0;
  if (success) trace(b, level, pos, 0);
  if (success && level + 1 < b->nlevels && __builtin_popcountll(prev) == 1)
    or_bm_clear(b, level + 1, cid);
  if (success) resolve_pending(b, level, pos, 1);
  return success;
}

/* try_set: symmetric, cascading set on set-first (Def. P:1129). */
int or_bm_try_set(or_bitmap_t* b, uint32_t level, uint64_t pos) {
  uint64_t cid = pos / b->W, mask = 1ULL << (pos % b->W);
  uint64_t prev = b->c[level][cid];
  b->c[level][cid] = prev | mask;
  int success = (prev & mask) == 0;
  if (success) trace(b, level, pos, 1);
  if (success && level + 1 < b->nlevels && prev == 0)
    or_bm_set(b, level + 1, cid);
  if (success) resolve_pending(b, level, pos, 0);
  return success;
}

/* clear(pos) == while (!try_clear(pos)) {}: an op that finds the bit
 * already cleared waits (pending) until a set of the same bit lets it
 * through; one still waiting at quiescence is the paper's deadlock (illegal
 * use), reported by or_bm_error. */
void or_bm_clear(or_bitmap_t* b, uint32_t level, uint64_t pos) {
  if (!or_bm_try_clear(b, level, pos)) add_pending(b, level, pos, 0);
}
void or_bm_set(or_bitmap_t* b, uint32_t level, uint64_t pos) {
  if (!or_bm_try_set(b, level, pos)) add_pending(b, level, pos, 1);
}

/* Alg. 4 (NoShift): cid from the nested bitmap, then ffs in container[cid]. */
int64_t or_bm_try_find_set(or_bitmap_t* b, uint32_t level) {
  uint64_t cid;
  if (level + 1 < b->nlevels) {
    int64_t r = or_bm_try_find_set(b, level + 1);
    if (r < 0) return -1;
    cid = (uint64_t)r;
  } else {
    cid = 0;
  }
  uint64_t c = b->c[level][cid] & wmask(b->W);
  if (c == 0) return -1;
  return (int64_t)(b->W * cid + (uint64_t)__builtin_ctzll(c));
}

/* clear(): "atomically clears and returns the position of an arbitrary set
 * bit"; loop find + try_clear until the clear succeeds or find FAILs. */
int64_t or_bm_clear_any(or_bitmap_t* b) {
  for (;;) {
    int64_t i = or_bm_try_find_set(b, 0);
    if (i < 0) return -1;
    if (or_bm_try_clear(b, 0, (uint64_t)i)) return i;
  }
}

int or_bm_get(const or_bitmap_t* b, uint64_t pos) {
  return (int)((b->c[0][pos / b->W] >> (pos % b->W)) & 1);
}

/* Alg. 5: selected <- nested.indices() (or [0]); for each selected container
 * append W*cid + nth_bit(c, i) for i < popc(c).  Sequential, so the output is
 * sorted; the paper's parallel version is unordered. */
uint64_t or_bm_indices(const or_bitmap_t* b, uint32_t level, uint64_t* out) {
  uint64_t nsel;
  uint64_t* sel;
  if (level + 1 < b->nlevels) {
    sel = (uint64_t*)malloc(sizeof(uint64_t) * (b->size[level + 1] + 1));
    nsel = or_bm_indices(b, level + 1, sel);
  } else {
    sel = (uint64_t*)malloc(sizeof(uint64_t));
    sel[0] = 0;
    nsel = 1;
  }
  uint64_t r = 0;
  for (uint64_t k = 0; k < nsel; k++) {
    uint64_t cid = sel[k];
    uint64_t c = b->c[level][cid];
    int pc = __builtin_popcountll(c);
    for (int i = 0; i < pc; i++) {
      /* nth_bit(c, i): b <- b & (b-1) applied i times, then ffs */
      uint64_t x = c;
      for (int j = 0; j < i; j++) x &= x - 1;
      out[r++] = b->W * cid + (uint64_t)__builtin_ctzll(x);
    }
  }
  free(sel);
  return r;
}

/* Definition: b_i^{l+1} = OR_k b^l_{W i + k} for every level. */
int or_bm_consistent(const or_bitmap_t* b) {
  for (uint32_t l = 0; l + 1 < b->nlevels; l++) {
    uint64_t nc = (b->size[l] + b->W - 1) / b->W;
    for (uint64_t i = 0; i < nc; i++) {
      int any = 0;
      for (uint32_t k = 0; k < b->W; k++)
        if ((b->c[l][i] >> k) & 1) any = 1;
      int up = (int)((b->c[l + 1][i / b->W] >> (i % b->W)) & 1);
      if (any != up) return 0;
    }
  }
  /* padding bits beyond size never set (reading R-PAD) */
  for (uint32_t l = 0; l < b->nlevels; l++) {
    uint64_t nc = (b->size[l] + b->W - 1) / b->W;
    for (uint64_t i = b->size[l]; i < nc * b->W; i++)
      if ((b->c[l][i / b->W] >> (i % b->W)) & 1) return 0;
  }
  return 1;
}

uint64_t or_bm_word(const or_bitmap_t* b, uint32_t level, uint64_t i) { return b->c[level][i]; }
uint32_t or_bm_nlevels(const or_bitmap_t* b) { return b->nlevels; }
uint64_t or_bm_level_words(const or_bitmap_t* b, uint32_t level) {
  return (b->size[level] + b->W - 1) / b->W;
}
void or_bm_trace(or_bitmap_t* b, int on) { b->trace_on = (uint32_t)on; b->ntrace = 0; }
uint32_t or_bm_ntrace(const or_bitmap_t* b) { return b->ntrace; }
void or_bm_trace_get(const or_bitmap_t* b, uint32_t i, uint32_t* lvl, uint32_t* pos, uint32_t* is_set) {
  *lvl = b->trace[i][0]; *pos = b->trace[i][1]; *is_set = b->trace[i][2];
}
int or_bm_error(const or_bitmap_t* b) { return b->error || b->npend > 0; }
