/*
 * oracle/wator.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Wa-Tor predator-prey (Table 1): "Fish/sharks occupy a 2D grid of
 * cells and can move to neighboring cells. Fish and sharks reproduce after
 * some iterations. Fish die when they are eaten and sharks starve to death
 * when they run out of food."  8 do-alls per iteration, classes Cell, Fish,
 * Shark (+ the Agent base, not materialised).  The per-pass rules, the
 * request/decide protocol and the counter-based RNG are reading R-WATOR
 * (SURVEY c.2 / C23), with Dewdney starvation (energy SS, -1 per step, reset
 * on eating).  Passes:
 *   1 Cell.prepare   2 Fish.prepare   3 Cell.decide   4 Fish.update
 *   5 Cell.prepare   6 Shark.prepare  7 Cell.decide   8 Shark.update
 * or_wator_dense runs the same rules on cell-indexed arrays (no objects).
 */
#include "store.h"

enum { K_EMPTY = 0, K_FISH = 1, K_SHARK = 2 };
enum { T_CELL = 3, T_FISH = 1, T_SHARK = 2 };
typedef struct { uint32_t id; uint64_t agent; uint8_t req[5]; } cell_rec;
typedef struct { uint32_t cell, target, egg; } fish_rec;
typedef struct { uint32_t cell, target, egg, energy; } shark_rec;

/* von Neumann neighbour d in {N,E,S,W} = 0..3 on the torus; opp(d) = d ^ 2 */
static uint32_t nbr4(uint32_t W, uint32_t H, uint32_t c, uint32_t d) {
  uint32_t x = c % W, y = c / W;
  switch (d) {
    case 0: y = (y + H - 1) % H; break;
    case 1: x = (x + 1) % W; break;
    case 2: y = (y + 1) % H; break;
    default: x = (x + W - 1) % W; break;
  }
  return y * W + x;
}
/* pick(list) = list[(key >> 32) % |list|] */
static uint32_t pick(const uint32_t* list, uint32_t n, uint64_t key) { return list[(key >> 32) % n]; }

typedef struct {
  uint32_t W, H, N;
  const or_wator_params_t* p;
  ost_t cells, fish, sharks;
  uint64_t* cell_h;        /* id -> Cell handle (from parallel_new order) */
  uint64_t born_f, born_s, eaten, starved;
  int err;
} wt_t;

static cell_rec* CR(wt_t* w, uint32_t c) { return (cell_rec*)ost_get(&w->cells, w->cell_h[c]); }

static void pass_cell_prepare(wt_t* w, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->cells, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) memset(((cell_rec*)ost_get(&w->cells, s[i]))->req, 0, 5);
  free(s);
}

static void pass_cell_decide(wt_t* w, uint32_t step, uint64_t phase, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->cells, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) {
    cell_rec* c = (cell_rec*)ost_get(&w->cells, s[i]);
    if (c->req[4]) continue;
    uint32_t D[4], nd = 0;
    for (uint32_t d = 0; d < 4; d++) if (c->req[d]) D[nd++] = d;
    if (!nd) continue;
    uint32_t d = pick(D, nd, or_key(w->p->seed, step, phase, c->id));
    uint64_t a = CR(w, nbr4(w->W, w->H, c->id, d))->agent;
    if (ost_htype(a) == T_FISH) ((fish_rec*)ost_get(&w->fish, a))->target = c->id;
    else if (ost_htype(a) == T_SHARK) ((shark_rec*)ost_get(&w->sharks, a))->target = c->id;
    else w->err |= 8;
  }
  free(s);
}

static void pass_fish_prepare(wt_t* w, uint32_t step, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->fish, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) {
    fish_rec* f = (fish_rec*)ost_get(&w->fish, s[i]);
    f->egg += 1;
    f->target = f->cell;
    uint32_t fr[4], nf = 0;
    for (uint32_t d = 0; d < 4; d++) if (CR(w, nbr4(w->W, w->H, f->cell, d))->agent == 0) fr[nf++] = d;
    if (nf) {
      uint32_t d = pick(fr, nf, or_key(w->p->seed, step, OR_PH_FISH_REQ, f->cell));
      CR(w, nbr4(w->W, w->H, f->cell, d))->req[d ^ 2] = 1;
    } else {
      CR(w, f->cell)->req[4] = 1;
    }
  }
  free(s);
}

static void pass_fish_update(wt_t* w, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->fish, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) {
    fish_rec* f = (fish_rec*)ost_get(&w->fish, s[i]);
    if (f->target == f->cell) continue;
    uint32_t old = f->cell;
    CR(w, old)->agent = 0;
    CR(w, f->target)->agent = s[i];
    f->cell = f->target;
    if (f->egg >= w->p->FB) {
      f->egg = 0;
      uint64_t h = ost_new(&w->fish);
      fish_rec* nf = (fish_rec*)ost_get(&w->fish, h);   /* f may move on realloc */
      nf->cell = old; nf->target = old; nf->egg = 0;
      CR(w, old)->agent = h;
      w->born_f++;
    }
  }
  free(s);
}

static void pass_shark_prepare(wt_t* w, uint32_t step, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->sharks, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) {
    shark_rec* k = (shark_rec*)ost_get(&w->sharks, s[i]);
    k->egg += 1;
    k->energy -= 1;
    k->target = k->cell;
    if (k->energy == 0) continue;                  /* starves in Shark.update */
    uint32_t fd[4], nfd = 0, fr[4], nfr = 0;
    for (uint32_t d = 0; d < 4; d++) {
      uint64_t a = CR(w, nbr4(w->W, w->H, k->cell, d))->agent;
      if (a && ost_htype(a) == T_FISH) fd[nfd++] = d;
      if (a == 0) fr[nfr++] = d;
    }
    uint64_t key = or_key(w->p->seed, step, OR_PH_SHARK_REQ, k->cell);
    if (nfd) {
      uint32_t d = pick(fd, nfd, key);
      CR(w, nbr4(w->W, w->H, k->cell, d))->req[d ^ 2] = 1;
    } else if (nfr) {
      uint32_t d = pick(fr, nfr, key);
      CR(w, nbr4(w->W, w->H, k->cell, d))->req[d ^ 2] = 1;
    } else {
      CR(w, k->cell)->req[4] = 1;
    }
  }
  free(s);
}

static void pass_shark_update(wt_t* w, uint64_t os, uint64_t salt) {
  uint64_t n, *s = ost_snapshot(&w->sharks, &n, os, salt);
  for (uint64_t i = 0; i < n; i++) {
    shark_rec* k = (shark_rec*)ost_get(&w->sharks, s[i]);
    if (k->energy == 0) {
      CR(w, k->cell)->agent = 0;
      w->err |= ost_destroy(&w->sharks, s[i]);       /* self-delete */
      w->starved++;
      continue;
    }
    if (k->target == k->cell) continue;
    uint64_t a = CR(w, k->target)->agent;
    if (a && ost_htype(a) == T_FISH) {
      w->err |= ost_destroy(&w->fish, a);            /* other type */
      k->energy = w->p->SS;
      w->eaten++;
    }
    uint32_t old = k->cell;
    CR(w, old)->agent = 0;
    CR(w, k->target)->agent = s[i];
    k->cell = k->target;
    if (k->egg >= w->p->SB) {
      k->egg = 0;
      uint64_t h = ost_new(&w->sharks);
      shark_rec* ns = (shark_rec*)ost_get(&w->sharks, h);
      ns->cell = old; ns->target = old; ns->egg = 0; ns->energy = w->p->SS;
      CR(w, old)->agent = h;
      w->born_s++;
    }
  }
  free(s);
}

int or_wator_run(uint32_t W, uint32_t H, uint8_t* kind, uint32_t* egg, uint32_t* energy,
                 const or_wator_params_t* p, uint32_t step0, uint32_t steps, uint64_t order_seed,
                 uint64_t* counters) {
  wt_t w;
  memset(&w, 0, sizeof(w));
  w.W = W; w.H = H; w.N = W * H; w.p = p;
  ost_init(&w.cells, T_CELL, sizeof(cell_rec));
  ost_init(&w.fish, T_FISH, sizeof(fish_rec));
  ost_init(&w.sharks, T_SHARK, sizeof(shark_rec));
  w.cell_h = (uint64_t*)malloc(sizeof(uint64_t) * w.N);
  /* parallel_new<Cell>(W*H): constructor i gets id i */
  for (uint32_t c = 0; c < w.N; c++) {
    uint64_t h = ost_new(&w.cells);
    ((cell_rec*)ost_get(&w.cells, h))->id = c;
    w.cell_h[c] = h;
  }
  for (uint32_t c = 0; c < w.N; c++) {
    if (kind[c] == K_FISH) {
      uint64_t h = ost_new(&w.fish);
      fish_rec* f = (fish_rec*)ost_get(&w.fish, h);
      f->cell = c; f->target = c; f->egg = egg[c];
      CR(&w, c)->agent = h;
    } else if (kind[c] == K_SHARK) {
      uint64_t h = ost_new(&w.sharks);
      shark_rec* k = (shark_rec*)ost_get(&w.sharks, h);
      k->cell = c; k->target = c; k->egg = egg[c]; k->energy = energy[c];
      CR(&w, c)->agent = h;
    }
  }
  for (uint32_t i = 0; i < steps; i++) {
    uint32_t step = step0 + i;
    uint64_t salt = 8ULL * step;
    w.born_f = w.born_s = w.eaten = w.starved = 0;
    pass_cell_prepare(&w, order_seed, salt + 0);
    pass_fish_prepare(&w, step, order_seed, salt + 1);
    pass_cell_decide(&w, step, OR_PH_FISH_DEC, order_seed, salt + 2);
    pass_fish_update(&w, order_seed, salt + 3);
    pass_cell_prepare(&w, order_seed, salt + 4);
    pass_shark_prepare(&w, step, order_seed, salt + 5);
    pass_cell_decide(&w, step, OR_PH_SHARK_DEC, order_seed, salt + 6);
    pass_shark_update(&w, order_seed, salt + 7);
    if (counters) {
      uint64_t* c = counters + 6ULL * i;
      c[0] = w.fish.nlive; c[1] = w.sharks.nlive; c[2] = w.born_f; c[3] = w.born_s;
      c[4] = w.eaten; c[5] = w.starved;
    }
  }
  /* canonical output: per cell (kind, egg, energy) */
  for (uint32_t c = 0; c < w.N; c++) {
    uint64_t a = CR(&w, c)->agent;
    kind[c] = K_EMPTY; egg[c] = 0; energy[c] = 0;
    if (a && ost_htype(a) == T_FISH) {
      fish_rec* f = (fish_rec*)ost_get(&w.fish, a);
      if (f->cell != c) w.err |= 16;
      kind[c] = K_FISH; egg[c] = f->egg;
    } else if (a && ost_htype(a) == T_SHARK) {
      shark_rec* k = (shark_rec*)ost_get(&w.sharks, a);
      if (k->cell != c) w.err |= 16;
      kind[c] = K_SHARK; egg[c] = k->egg; energy[c] = k->energy;
    }
  }
  free(w.cell_h);
  ost_fini(&w.cells); ost_fini(&w.fish); ost_fini(&w.sharks);
  return w.err;
}

/* ---- dense-grid reformulation: same rules on cell-indexed arrays ---- */
int or_wator_dense(uint32_t W, uint32_t H, uint8_t* kind, uint32_t* egg, uint32_t* energy,
                   const or_wator_params_t* p, uint32_t step0, uint32_t steps, uint64_t* counters) {
  uint32_t N = W * H;
  uint8_t* req = (uint8_t*)malloc(5ULL * N);
  uint32_t* target = (uint32_t*)malloc(sizeof(uint32_t) * N);   /* indexed by the agent's cell */
  uint32_t* list = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (uint32_t i = 0; i < steps; i++) {
    uint32_t step = step0 + i;
    uint64_t born_f = 0, born_s = 0, eaten = 0, starved = 0;
    for (int half = 0; half < 2; half++) {
      uint8_t me = half == 0 ? K_FISH : K_SHARK;
      memset(req, 0, 5ULL * N);
      uint32_t nl = 0;
      for (uint32_t c = 0; c < N; c++) if (kind[c] == me) list[nl++] = c;   /* snapshot */
      /* prepare */
      for (uint32_t j = 0; j < nl; j++) {
        uint32_t c = list[j];
        egg[c] += 1;
        target[c] = c;
        if (me == K_SHARK) { energy[c] -= 1; if (energy[c] == 0) continue; }
        uint32_t fd[4], nfd = 0, fr[4], nfr = 0;
        for (uint32_t d = 0; d < 4; d++) {
          uint32_t e = nbr4(W, H, c, d);
          if (kind[e] == K_FISH) fd[nfd++] = d;
          if (kind[e] == K_EMPTY) fr[nfr++] = d;
        }
        uint64_t key = or_key(p->seed, step, me == K_FISH ? OR_PH_FISH_REQ : OR_PH_SHARK_REQ, c);
        int d = -1;
        if (me == K_SHARK && nfd) d = (int)pick(fd, nfd, key);
        else if (nfr) d = (int)pick(fr, nfr, key);
        if (d >= 0) req[5ULL * nbr4(W, H, c, (uint32_t)d) + ((uint32_t)d ^ 2)] = 1;
        else req[5ULL * c + 4] = 1;
      }
      /* decide */
      for (uint32_t c = 0; c < N; c++) {
        if (req[5ULL * c + 4]) continue;
        uint32_t D[4], nd = 0;
        for (uint32_t d = 0; d < 4; d++) if (req[5ULL * c + d]) D[nd++] = d;
        if (!nd) continue;
        uint32_t d = pick(D, nd, or_key(p->seed, step, me == K_FISH ? OR_PH_FISH_DEC : OR_PH_SHARK_DEC, c));
        target[nbr4(W, H, c, d)] = c;
      }
      /* update: move the snapshot agents (state travels with the agent) */
      for (uint32_t j = 0; j < nl; j++) {
        uint32_t c = list[j];
        if (me == K_SHARK && energy[c] == 0) {
          kind[c] = K_EMPTY; egg[c] = 0; energy[c] = 0; starved++;
          continue;
        }
        uint32_t t = target[c];
        if (t == c) continue;
        uint32_t e_egg = egg[c], e_en = energy[c];
        if (me == K_SHARK && kind[t] == K_FISH) { eaten++; e_en = p->SS; }
        kind[c] = K_EMPTY; egg[c] = 0; energy[c] = 0;
        kind[t] = me; egg[t] = e_egg; energy[t] = e_en;
        if (e_egg >= (me == K_FISH ? p->FB : p->SB)) {
          egg[t] = 0;
          kind[c] = me; egg[c] = 0; energy[c] = me == K_SHARK ? p->SS : 0;
          if (me == K_FISH) born_f++; else born_s++;
        }
      }
    }
    if (counters) {
      uint64_t nf = 0, ns = 0;
      for (uint32_t c = 0; c < N; c++) { nf += kind[c] == K_FISH; ns += kind[c] == K_SHARK; }
      uint64_t* q = counters + 6ULL * i;
      q[0] = nf; q[1] = ns; q[2] = born_f; q[3] = born_s; q[4] = eaten; q[5] = starved;
    }
  }
  free(req); free(target); free(list);
  return 0;
}
