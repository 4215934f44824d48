/*
 * oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the DynaSOAr hot path
 * (Springer & Masuhara, arXiv 1810.11765; "P:n" = line n of PAPER.md).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code with
 * paper_1810_11765_b200/csrc (the CUDA path) and includes nothing from it.
 *
 * Every function cites the passage it follows.  Where the paper is silent or
 * garbled we follow the reading listed in DESIGN.md ("R-xx" ids there; the
 * SURVEY.md §8(c) ids "Cnn" are quoted beside them).
 */
#ifndef DSR_ORACLE_H
#define DSR_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- counter-based RNG (SURVEY c.5; SplitMix64 mixer) --------- */
uint64_t or_sm(uint64_t x);
uint64_t or_key(uint64_t seed, uint64_t step, uint64_t phase, uint64_t idx);
enum { OR_PH_INIT = 0, OR_PH_FISH_REQ = 1, OR_PH_FISH_DEC = 2,
       OR_PH_SHARK_REQ = 3, OR_PH_SHARK_DEC = 4, OR_PH_MB_FIELD = 5 };

/* ---------------- heap layout (reading R-LAYOUT) -- */
#define OR_MAXT 8
#define OR_MAXF 16
#define OR_MAXL 8
typedef struct {
  uint32_t ntypes;
  uint32_t nfields[OR_MAXT];
  uint32_t fsize[OR_MAXT][OR_MAXF];
  uint32_t cap[OR_MAXT];                 /* N_T, eq. P:308 */
  uint32_t col_off[OR_MAXT][OR_MAXF];    /* byte offset of field column (R-LAYOUT) */
  uint32_t block_bytes;                  /* data-segment bytes per block */
  uint64_t M;                            /* upper bound on the block count (see or_layout) */
  uint32_t nlevels;                      /* levels of one M-bit bitmap */
  uint64_t level_words[OR_MAXL];         /* u64 containers per level */
} or_layout_t;

/* returns 0 on success, nonzero on invalid input (type > 64x smallest, ...) */
int or_layout(uint32_t ntypes, const uint32_t* nfields, const uint32_t* fsizes_flat,
              uint64_t heap_bytes, or_layout_t* out);

/* ---------------- hierarchical bitmap, container width W ------- */
typedef struct {
  uint64_t n;            /* leaf bits N */
  uint32_t W;            /* container width (64 in DynaSOAr; 4 in Fig. 7) */
  uint32_t nlevels;
  uint64_t size[OR_MAXL];   /* bits per level */
  uint64_t* c[OR_MAXL];     /* containers per level (W low bits used) */
  /* trace of set/clear operations performed (level, pos, is_set) for pins */
  uint32_t trace_on, ntrace;
  uint32_t trace[64][3];
  int error;             /* set on illegal use (spin-forever in the paper) */
  /* set / clear ops that found their bit already in the target state: the
   * paper's op "spins until it actually changed the bit";
   * sequentially it waits here and completes right after the opposite op on
   * the same bit.  Still pending at quiescence = the paper's deadlock. */
  uint32_t npend;
  uint32_t pend_lvl[16], pend_set[16];
  uint64_t pend_pos[16];
} or_bitmap_t;

or_bitmap_t* or_bm_new(uint64_t n, uint32_t W, int all_set);
void or_bm_free(or_bitmap_t* b);
int or_bm_try_set(or_bitmap_t* b, uint32_t level, uint64_t pos);
int or_bm_try_clear(or_bitmap_t* b, uint32_t level, uint64_t pos);
void or_bm_set(or_bitmap_t* b, uint32_t level, uint64_t pos);
void or_bm_clear(or_bitmap_t* b, uint32_t level, uint64_t pos);
int64_t or_bm_try_find_set(or_bitmap_t* b, uint32_t level);
int64_t or_bm_clear_any(or_bitmap_t* b);
int or_bm_get(const or_bitmap_t* b, uint64_t pos);
uint64_t or_bm_indices(const or_bitmap_t* b, uint32_t level, uint64_t* out);
int or_bm_consistent(const or_bitmap_t* b);
uint64_t or_bm_word(const or_bitmap_t* b, uint32_t level, uint64_t i);
uint32_t or_bm_nlevels(const or_bitmap_t* b);
uint64_t or_bm_level_words(const or_bitmap_t* b, uint32_t level);
void or_bm_trace(or_bitmap_t* b, int on);
uint32_t or_bm_ntrace(const or_bitmap_t* b);
void or_bm_trace_get(const or_bitmap_t* b, uint32_t i, uint32_t* lvl, uint32_t* pos, uint32_t* is_set);
int or_bm_error(const or_bitmap_t* b);

/* ---------------- sequential model of the paper's heap (Algs. 1-9) --------- */
typedef struct or_heap or_heap_t;
/* a heap of exactly M blocks ("M is determined at compile time") */
or_heap_t* or_heap_new(uint32_t ntypes, const uint32_t* nfields, const uint32_t* fsizes_flat, uint64_t M);
void or_heap_free(or_heap_t* h);
uint64_t or_heap_alloc(or_heap_t* h, uint32_t type);      /* 0 == OOM */
int or_heap_dealloc(or_heap_t* h, uint64_t handle);       /* 0 ok */
uint64_t or_heap_M(const or_heap_t* h);
uint64_t or_heap_alloc_bm(const or_heap_t* h, uint64_t bid);
uint32_t or_heap_type(const or_heap_t* h, uint64_t bid);
/* which: 0 = free, 1 = allocated[t], 2 = active[t] */
or_bitmap_t* or_heap_bitmap(or_heap_t* h, uint32_t which, uint32_t type);
uint64_t or_heap_live(const or_heap_t* h, uint32_t type);
double or_heap_fragmentation(const or_heap_t* h);
int or_heap_error(const or_heap_t* h);
/* Scripted interleavings (pins of the concurrent branches of Algs. 1, 2, 9):
 * a one-shot hook called at a linearisation point, from which the test runs
 * "another thread's" operations on the same heap.
 *   OR_HOOK_FOUND        or_heap_alloc: block bid chosen (active or fresh), before the reservation (Alg. 1 l.9)
 *   OR_HOOK_EMPTIED      dealloc: the last slot of bid freed (EMPTY), before invalidate (Alg. 2 l.7)
 *   OR_HOOK_INVALIDATED  invalidate: atomicOr(~0) returned before != pad, before the rollback (Alg. 9 l.8) */
enum { OR_HOOK_FOUND = 0, OR_HOOK_EMPTIED = 1, OR_HOOK_INVALIDATED = 2 };
typedef void (*or_hook_fn)(void* ctx, uint32_t point, uint64_t bid);
void or_heap_set_hook(or_heap_t* h, or_hook_fn fn, void* ctx, uint32_t point);
/* counters: 0 type-change rollbacks (Alg. 1 l.14), 1 failed invalidations
 * (Alg. 9 l.8), 2 invalidation retries after an empty-again rollback (l.12),
 * 3 deferred deactivations (l.10) */
uint64_t or_heap_counter(const or_heap_t* h, uint32_t k);

/* handle codec, Fig. 5 / Listing 2, readings C6/C7 */
uint64_t or_handle_encode(uint32_t type, uint32_t cap, uint64_t bid, uint32_t slot);
void or_handle_decode(uint64_t h, uint32_t* type, uint32_t* cap, uint64_t* bid, uint32_t* slot);

/* thread assignment, reading C9 (element stride) */
uint64_t or_assign_num_blocks(uint64_t r, uint32_t NT, uint64_t n, uint64_t tid);
uint64_t or_assign_block_pos(uint32_t NT, uint64_t n, uint64_t tid, uint64_t k);  /* index into R */
uint32_t or_assign_slot(uint32_t NT, uint64_t n, uint64_t tid, uint64_t k);

/* ---------------- SMMO workloads on a plain object store ------------------- */
/* microbench (SURVEY c.4).  out[0..17]: phase 2 (count,sum,xor) for A,B,C then
 * phase 5 (count,sum,xor) for A,B,C.  live_out[0..3*6-1]: live(A,B,C) after
 * each phase 1..6.  order_seed != 0 shuffles every do-all's visit order. */
int or_microbench(uint64_t seed, uint64_t n1, uint64_t n2, uint64_t order_seed,
                  uint64_t* out, uint64_t* live_out);
int or_microbench_live(uint64_t seed, uint64_t n1, uint64_t n2, uint32_t stop, uint32_t ty,
                       uint32_t* out, uint64_t cap, uint64_t* count);

/* Game of Life, O(#alive) Alive/Candidate version (SURVEY c.1, Table 1).
 * alive: W*H bytes (0/1), updated in place after `gens` generations.
 * dump_every: if nonzero, per-generation canonical records are appended to
 * dump (records of 4 u32: cell, kind(1 alive,2 cand), is_new, action), with
 * per-generation counts in dump_counts[g].  Returns 0 on success. */
int or_gol_run(uint32_t W, uint32_t H, uint8_t* alive, uint32_t gens, uint64_t order_seed,
               uint32_t* dump, uint64_t dump_cap, uint64_t* dump_counts);
/* Dense B3/S23 Life on a torus (textbook). */
void or_life_dense(uint32_t W, uint32_t H, uint8_t* alive, uint32_t gens);

/* Wa-Tor (SURVEY c.2, Table 1).  kind: 0 empty, 1 fish, 2 shark. */
typedef struct { uint32_t FB, SB, SS; uint64_t seed; } or_wator_params_t;
int or_wator_run(uint32_t W, uint32_t H, uint8_t* kind, uint32_t* egg, uint32_t* energy,
                 const or_wator_params_t* p, uint32_t step0, uint32_t steps, uint64_t order_seed,
                 uint64_t* counters /* steps x 6: fish, sharks, fish_born, shark_born, eaten, starved */);
int or_wator_dense(uint32_t W, uint32_t H, uint8_t* kind, uint32_t* egg, uint32_t* energy,
                   const or_wator_params_t* p, uint32_t step0, uint32_t steps, uint64_t* counters);

/* N-body with collisions (SURVEY c.3, Listing 1, Table 1). */
typedef struct { double G, dt, eps, R; int merges; } or_nbody_params_t;
/* state arrays of length n (fp32 stored, fp64 arithmetic); alive[i] 0/1. */
int or_nbody_run(uint32_t n, float* x, float* y, float* vx, float* vy, float* m,
                 uint8_t* alive, const or_nbody_params_t* p, uint32_t steps);

#ifdef __cplusplus
}
#endif
#endif
