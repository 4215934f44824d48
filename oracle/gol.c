/*
 * oracle/gol.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Game of Life with O(#alive) work (Table 1): "Cells can be dead,
 * alive or alive-candidates. Alive-candidates are dead cells that may become
 * active in the next iteration. Only alive-candidates and alive cells are
 * processed with parallel do-all operations."  4 do-alls per iteration,
 * dynamic classes Alive and Candidate.  The per-pass rules are reading
 * R-GOL (SURVEY c.1 / C22): torus, Moore neighbourhood, rule B3/S23.
 *   pass 1 Candidate.prepare : k = #Alive neighbours (type from handle bits,
 *                              P:333); k == 3 -> SPAWN, k == 0 -> DIE
 *   pass 2 Alive.prepare     : is_new = 0; k < 2 or k > 3 -> DIE
 *   pass 3 Candidate.update  : SPAWN -> destroy(this), cell = new Alive(is_new=1);
 *                              DIE -> destroy(this), cell = empty
 *   pass 4 Alive.update      : is_new -> every empty neighbour gets a new
 *                              Candidate (exactly one); old and DIE ->
 *                              destroy(this), cell = new Candidate
 * plus the textbook dense Life that pins it.
 */
#include "store.h"

enum { GOL_ALIVE = 1, GOL_CAND = 2 };
enum { ACT_NONE = 0, ACT_SPAWN = 1, ACT_DIE = 2 };
typedef struct { uint32_t cell; uint8_t is_new, action; } alive_rec;
typedef struct { uint32_t cell; uint8_t action; } cand_rec;

static uint32_t nbr8(uint32_t W, uint32_t H, uint32_t c, int k) {
  static const int dx[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
  static const int dy[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  uint32_t x = c % W, y = c / W;
  uint32_t nx = (x + W + (uint32_t)(dx[k] + 1) - 1) % W;
  uint32_t ny = (y + H + (uint32_t)(dy[k] + 1) - 1) % H;
  return ny * W + nx;
}

static uint32_t count_alive(const uint64_t* cell, uint32_t W, uint32_t H, uint32_t c) {
  uint32_t k = 0;
  for (int d = 0; d < 8; d++) {
    uint64_t h = cell[nbr8(W, H, c, d)];
    if (h && ost_htype(h) == GOL_ALIVE) k++;
  }
  return k;
}

static uint64_t dump_gen(ost_t* A, ost_t* C, uint32_t N, const uint64_t* cell, uint32_t* out) {
  /* canonical records sorted by cell (each cell holds <= 1 object) */
  uint64_t k = 0;
  for (uint32_t c = 0; c < N; c++) {
    uint64_t h = cell[c];
    if (!h) continue;
    if (ost_htype(h) == GOL_ALIVE) {
      alive_rec* a = (alive_rec*)ost_get(A, h);
      out[4 * k + 0] = a->cell; out[4 * k + 1] = GOL_ALIVE; out[4 * k + 2] = a->is_new; out[4 * k + 3] = a->action;
    } else {
      cand_rec* q = (cand_rec*)ost_get(C, h);
      out[4 * k + 0] = q->cell; out[4 * k + 1] = GOL_CAND; out[4 * k + 2] = 0; out[4 * k + 3] = q->action;
    }
    k++;
  }
  return k;
}

int or_gol_run(uint32_t W, uint32_t H, uint8_t* alive, uint32_t gens, uint64_t order_seed,
               uint32_t* dump, uint64_t dump_cap, uint64_t* dump_counts) {
  uint32_t N = W * H;
  uint64_t* cell = (uint64_t*)calloc(N, sizeof(uint64_t));
  ost_t A, C;
  ost_init(&A, GOL_ALIVE, sizeof(alive_rec));
  ost_init(&C, GOL_CAND, sizeof(cand_rec));
  int err = 0;
  /* initial state: Alive(c) for alive cells, Candidate(c) for dead cells with
   * >= 1 alive neighbour (the Candidate invariant) */
  for (uint32_t c = 0; c < N; c++)
    if (alive[c]) {
      uint64_t h = ost_new(&A);
      alive_rec* a = (alive_rec*)ost_get(&A, h);
      a->cell = c; a->is_new = 0; a->action = ACT_NONE;
      cell[c] = h;
    }
  for (uint32_t c = 0; c < N; c++)
    if (!alive[c] && count_alive(cell, W, H, c) > 0) {
      uint64_t h = ost_new(&C);
      cand_rec* q = (cand_rec*)ost_get(&C, h);
      q->cell = c; q->action = ACT_NONE;
      cell[c] = h;
    }
  uint64_t used = 0;
  for (uint32_t g = 0; g < gens; g++) {
    uint64_t n, *s;
    /* pass 1: Candidate.prepare */
    s = ost_snapshot(&C, &n, order_seed, 4ULL * g + 0);
    for (uint64_t i = 0; i < n; i++) {
      cand_rec* q = (cand_rec*)ost_get(&C, s[i]);
      uint32_t k = count_alive(cell, W, H, q->cell);
      q->action = k == 3 ? ACT_SPAWN : (k == 0 ? ACT_DIE : ACT_NONE);
    }
    free(s);
    /* pass 2: Alive.prepare */
    s = ost_snapshot(&A, &n, order_seed, 4ULL * g + 1);
    for (uint64_t i = 0; i < n; i++) {
      alive_rec* a = (alive_rec*)ost_get(&A, s[i]);
      uint32_t k = count_alive(cell, W, H, a->cell);
      a->is_new = 0;
      a->action = (k < 2 || k > 3) ? ACT_DIE : ACT_NONE;
    }
    free(s);
    /* pass 3: Candidate.update */
    s = ost_snapshot(&C, &n, order_seed, 4ULL * g + 2);
    for (uint64_t i = 0; i < n; i++) {
      cand_rec* q = (cand_rec*)ost_get(&C, s[i]);
      uint32_t c = q->cell;
      uint8_t act = q->action;
      if (act == ACT_SPAWN) {
        err |= ost_destroy(&C, s[i]);
        uint64_t h = ost_new(&A);
        alive_rec* a = (alive_rec*)ost_get(&A, h);
        a->cell = c; a->is_new = 1; a->action = ACT_NONE;
        cell[c] = h;
      } else if (act == ACT_DIE) {
        err |= ost_destroy(&C, s[i]);
        cell[c] = 0;
      }
    }
    free(s);
    /* pass 4: Alive.update */
    s = ost_snapshot(&A, &n, order_seed, 4ULL * g + 3);
    for (uint64_t i = 0; i < n; i++) {
      alive_rec* a = (alive_rec*)ost_get(&A, s[i]);
      uint32_t c = a->cell;
      if (a->is_new) {
        for (int d = 0; d < 8; d++) {
          uint32_t e = nbr8(W, H, c, d);
          if (cell[e] == 0) {
            uint64_t h = ost_new(&C);
            cand_rec* q = (cand_rec*)ost_get(&C, h);
            q->cell = e; q->action = ACT_NONE;
            cell[e] = h;
          }
        }
      } else if (a->action == ACT_DIE) {
        err |= ost_destroy(&A, s[i]);
        uint64_t h = ost_new(&C);
        cand_rec* q = (cand_rec*)ost_get(&C, h);
        q->cell = c; q->action = ACT_NONE;
        cell[c] = h;
      }
    }
    free(s);
    if (dump) {
      if (used + A.nlive + C.nlive > dump_cap) { err |= 4; break; }
      uint64_t k = dump_gen(&A, &C, N, cell, dump + 4 * used);
      dump_counts[g] = k;
      used += k;
    }
  }
  for (uint32_t c = 0; c < N; c++) alive[c] = (cell[c] && ost_htype(cell[c]) == GOL_ALIVE) ? 1 : 0;
  free(cell);
  ost_fini(&A);
  ost_fini(&C);
  return err;
}

/* Textbook dense Life, rule B3/S23 on a W x H torus. */
void or_life_dense(uint32_t W, uint32_t H, uint8_t* alive, uint32_t gens) {
  uint32_t N = W * H;
  uint8_t* nxt = (uint8_t*)malloc(N);
  for (uint32_t g = 0; g < gens; g++) {
    for (uint32_t y = 0; y < H; y++)
      for (uint32_t x = 0; x < W; x++) {
        int k = 0;
        for (int dy = -1; dy <= 1; dy++)
          for (int dx = -1; dx <= 1; dx++) {
            if (!dx && !dy) continue;
            uint32_t xx = (x + W + (uint32_t)dx) % W, yy = (y + H + (uint32_t)dy) % H;
            k += alive[yy * W + xx];
          }
        uint8_t a = alive[y * W + x];
        nxt[y * W + x] = (uint8_t)(k == 3 || (a && k == 2));
      }
    memcpy(alive, nxt, N);
  }
  free(nxt);
}
