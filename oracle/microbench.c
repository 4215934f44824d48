/*
 * oracle/microbench.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Allocator microbenchmark (BASELINE.json configs[4]; phases per SURVEY c.4),
 * written on the plain object store O1:
 *   types A{3 x u32}, B{4 x u32}, C{6 x u32}
 *   1. thread t < n1 does new [A,A,B,C][t & 3] and writes field k =
 *      low32(key(seed, 0, MB_FIELD, 16 t + k))           (device new)
 *   2. do-all per type: (count, sum of fields mod 2^64, xor of fields)
 *   3. do-all per type: if field0 & 1: destroy(this)     (self-delete)
 *   4. threads t' = n1 + t, t < n2, repeat phase 1
 *   5. reduce again
 *   6. do-all per type: destroy(this)                     (drain)
 */
#include "store.h"

static const uint32_t MB_NF[3] = {3, 4, 6};
static uint32_t mb_type(uint64_t t) { uint32_t q = (uint32_t)(t & 3); return q < 2 ? 0 : (q == 2 ? 1 : 2); }

static void mb_new_range(ost_t* st, uint64_t seed, uint64_t t0, uint64_t n) {
  for (uint64_t t = t0; t < t0 + n; t++) {
    uint32_t ty = mb_type(t);
    uint64_t h = ost_new(&st[ty]);
    uint32_t* f = (uint32_t*)ost_get(&st[ty], h);
    for (uint32_t k = 0; k < MB_NF[ty]; k++)
      f[k] = (uint32_t)or_key(seed, 0, OR_PH_MB_FIELD, t * 16 + k);
  }
}

static void mb_reduce(ost_t* st, uint64_t order_seed, uint64_t salt, uint64_t* out) {
  for (uint32_t ty = 0; ty < 3; ty++) {
    uint64_t n, cnt = 0, sum = 0, x = 0;
    uint64_t* snap = ost_snapshot(&st[ty], &n, order_seed, salt + ty);
    for (uint64_t i = 0; i < n; i++) {
      uint32_t* f = (uint32_t*)ost_get(&st[ty], snap[i]);
      cnt++;
      for (uint32_t k = 0; k < MB_NF[ty]; k++) { sum += f[k]; x ^= f[k]; }
    }
    free(snap);
    out[3 * ty + 0] = cnt;
    out[3 * ty + 1] = sum;
    out[3 * ty + 2] = x;
  }
}

static int mb_free_pass(ost_t* st, uint64_t order_seed, uint64_t salt, int odd_only) {
  int err = 0;
  for (uint32_t ty = 0; ty < 3; ty++) {
    uint64_t n;
    uint64_t* snap = ost_snapshot(&st[ty], &n, order_seed, salt + ty);
    for (uint64_t i = 0; i < n; i++) {
      uint32_t* f = (uint32_t*)ost_get(&st[ty], snap[i]);
      if (!odd_only || (f[0] & 1)) err |= ost_destroy(&st[ty], snap[i]);
    }
    free(snap);
  }
  return err;
}

int or_microbench(uint64_t seed, uint64_t n1, uint64_t n2, uint64_t order_seed,
                  uint64_t* out, uint64_t* live_out) {
  ost_t st[3];
  for (uint32_t ty = 0; ty < 3; ty++) ost_init(&st[ty], ty + 1, 4 * MB_NF[ty]);
  int err = 0;
#define LIVE(ph) do { for (int q = 0; q < 3; q++) live_out[3 * (ph) + q] = st[q].nlive; } while (0)
  mb_new_range(st, seed, 0, n1);                  LIVE(0);
  mb_reduce(st, order_seed, 100, out);            LIVE(1);
  err |= mb_free_pass(st, order_seed, 200, 1);    LIVE(2);
  mb_new_range(st, seed, n1, n2);                 LIVE(3);
  mb_reduce(st, order_seed, 300, out + 9);        LIVE(4);
  err |= mb_free_pass(st, order_seed, 400, 0);    LIVE(5);
#undef LIVE
  for (uint32_t ty = 0; ty < 3; ty++) ost_fini(&st[ty]);
  return err;
}

/* The live objects of type `ty` after phase `stop` (1 = after the first
 * allocation burst, 3 = after the odd-free pass, 4 = after the second burst),
 * each as its packed u32 fields in store order (the caller sorts them into the
 * canonical order, SURVEY c.8).  *count = live objects; records are written
 * only while they fit in cap u32 words.  Returns 1 on an illegal delete. */
int or_microbench_live(uint64_t seed, uint64_t n1, uint64_t n2, uint32_t stop, uint32_t ty,
                       uint32_t* out, uint64_t cap, uint64_t* count) {
  ost_t st[3];
  for (uint32_t q = 0; q < 3; q++) ost_init(&st[q], q + 1, 4 * MB_NF[q]);
  int err = 0;
  uint64_t scratch[9];
  mb_new_range(st, seed, 0, n1);
  if (stop >= 3) {
    mb_reduce(st, 0, 100, scratch);
    err |= mb_free_pass(st, 0, 200, 1);
  }
  if (stop >= 4) mb_new_range(st, seed, n1, n2);
  uint64_t k = 0;
  for (uint64_t i = 0; i < st[ty].n; i++) {
    if (!st[ty].live[i]) continue;
    if ((k + 1) * MB_NF[ty] <= cap) memcpy(out + k * MB_NF[ty], st[ty].data + i * st[ty].rec, st[ty].rec);
    k++;
  }
  *count = k;
  for (uint32_t q = 0; q < 3; q++) ost_fini(&st[q]);
  return err;
}
