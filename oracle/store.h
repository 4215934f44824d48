/*
 * oracle/store.h -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * O1: the plain object store the SMMO apps run on.  It is the "plain
 * definition" of the paper's programming interface:
 *   new / destroy
 *   parallel_do<T, f>             P:123  -- f runs on every object of T that
 *                                 exists at launch time; objects created during
 *                                 the pass are not visited (snapshot)
 *   parallel_new<T>(n)            P:124  -- n constructors with ids 0..n-1
 * Handles are (type << 32) | (index + 1); 0 is null.  Placement is irrelevant
 * to every result the apps report (reading R-CANON / C16).
 */
#ifndef DSR_ORACLE_STORE_H
#define DSR_ORACLE_STORE_H
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

typedef struct {
  uint32_t type;       /* app type id stored in the handle */
  uint32_t rec;        /* record bytes */
  uint64_t n, cap;     /* records in use / allocated */
  uint8_t* data;
  uint8_t* live;
  uint32_t* fl;        /* free list */
  uint64_t nfl;
  uint64_t nlive;
} ost_t;

static inline void ost_init(ost_t* s, uint32_t type, uint32_t rec) {
  memset(s, 0, sizeof(*s));
  s->type = type;
  s->rec = rec;
}
static inline void ost_fini(ost_t* s) { free(s->data); free(s->live); free(s->fl); memset(s, 0, sizeof(*s)); }

static inline uint64_t ost_new(ost_t* s) {
  uint64_t id;
  if (s->nfl) {
    id = s->fl[--s->nfl];
  } else {
    if (s->n == s->cap) {
      uint64_t nc = s->cap ? s->cap * 2 : 1024;
      s->data = (uint8_t*)realloc(s->data, nc * s->rec);
      s->live = (uint8_t*)realloc(s->live, nc);
      s->fl = (uint32_t*)realloc(s->fl, nc * sizeof(uint32_t));
      s->cap = nc;
    }
    id = s->n++;
  }
  s->live[id] = 1;
  memset(s->data + id * s->rec, 0, s->rec);
  s->nlive++;
  return ((uint64_t)s->type << 32) | (id + 1);
}
static inline uint64_t ost_id(uint64_t h) { return (h & 0xFFFFFFFFULL) - 1; }
static inline uint32_t ost_htype(uint64_t h) { return (uint32_t)(h >> 32); }
static inline void* ost_get(ost_t* s, uint64_t h) { return s->data + ost_id(h) * s->rec; }
static inline int ost_destroy(ost_t* s, uint64_t h) {
  uint64_t id = ost_id(h);
  if (ost_htype(h) != s->type || id >= s->n || !s->live[id]) return 1;   /* illegal delete */
  s->live[id] = 0;
  s->fl[s->nfl++] = (uint32_t)id;
  s->nlive--;
  return 0;
}

/* Snapshot of the live handles at pass start.  With
 * order_seed != 0 the visit order is a seeded permutation (the
 * "permutation test": results must not depend on it). */
static inline uint64_t* ost_snapshot(ost_t* s, uint64_t* count, uint64_t order_seed, uint64_t salt) {
  uint64_t* v = (uint64_t*)malloc((s->nlive + 1) * sizeof(uint64_t));
  uint64_t k = 0;
  for (uint64_t i = 0; i < s->n; i++)
    if (s->live[i]) v[k++] = ((uint64_t)s->type << 32) | (i + 1);
  if (order_seed) {
    for (uint64_t i = k; i > 1; i--) {
      uint64_t j = or_key(order_seed, salt, 7, i) % i;
      uint64_t t = v[i - 1]; v[i - 1] = v[j]; v[j] = t;
    }
  }
  *count = k;
  return v;
}
#endif
