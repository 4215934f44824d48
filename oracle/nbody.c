/*
 * oracle/nbody.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * N-body with collisions (Table 1: "particles are merged according to
 * perfectly inelastic collision when they are getting too close"; Listing 1
 * P:143-183; Fig. 1 caption P:42 / footnote P:46).  Reading R-NBODY
 * (SURVEY c.3, C24/C25/C28): six do-alls per step,
 *   1 compute_force  f_i = sum_{j != i} G m_i m_j (p_j - p_i) / (|p_j - p_i|^2 + eps^2)^{3/2}
 *                    (device_do over the snapshot S0; Plummer eps)
 *   2 move           v += f / m dt; p += v dt (velocity first)
 *   3 prepare_merge  target_i = argmin over j with (m_j, id_j) >lex (m_i, id_i)
 *                    and d2_ij < R^2 of (d2_ij, id_j), over the snapshot S1
 *   4 claim          incoming[target_i] = min(incoming, id_i)
 *   5 absorb         if incoming != NONE and target == NONE: m' = m + m_i
 *                    (fp32 add), v' = (m v + m_i v_i) / m', p' = (m p + m_i p_i) / m',
 *                    merged[i] = 1
 *   6 delete_merged  destroy bodies with merged = 1
 * State is stored in fp32 (like the GPU); arithmetic inside a pass is fp64.
 * merges = 0 gives the plain N-Body app (2 do-alls).
 * Bodies are indexed by id (the snapshot is id-indexed; dead ids have m = 0).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NONE 0xFFFFFFFFu

int or_nbody_run(uint32_t n, float* x, float* y, float* vx, float* vy, float* m,
                 uint8_t* alive, const or_nbody_params_t* p, uint32_t steps) {
  float* fx = (float*)calloc(n, sizeof(float));
  float* fy = (float*)calloc(n, sizeof(float));
  uint32_t* target = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* incoming = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint8_t* merged = (uint8_t*)calloc(n, 1);
  /* snapshot S (id-indexed, fp32 values as stored) */
  float* sx = (float*)malloc(sizeof(float) * n);
  float* sy = (float*)malloc(sizeof(float) * n);
  float* sm = (float*)malloc(sizeof(float) * n);
  float* svx = (float*)malloc(sizeof(float) * n);
  float* svy = (float*)malloc(sizeof(float) * n);
  double eps2 = p->eps * p->eps, R2 = p->R * p->R;
  for (uint32_t s = 0; s < steps; s++) {
    /* S0 */
    for (uint32_t i = 0; i < n; i++) { sx[i] = x[i]; sy[i] = y[i]; sm[i] = alive[i] ? m[i] : 0.0f; }
    /* pass 1: compute_force */
    for (uint32_t i = 0; i < n; i++) {
      if (!alive[i]) continue;
      double ax = 0.0, ay = 0.0;
      for (uint32_t j = 0; j < n; j++) {
        if (j == i || sm[j] == 0.0f) continue;
        double dx = (double)sx[j] - (double)sx[i], dy = (double)sy[j] - (double)sy[i];
        double r2 = dx * dx + dy * dy + eps2;
        double inv = 1.0 / (r2 * sqrt(r2));
        double F = p->G * (double)m[i] * (double)sm[j] * inv;
        ax += F * dx;
        ay += F * dy;
      }
      fx[i] = (float)ax;
      fy[i] = (float)ay;
    }
    /* pass 2: move */
    for (uint32_t i = 0; i < n; i++) {
      if (!alive[i]) continue;
      vx[i] = (float)((double)vx[i] + (double)fx[i] / (double)m[i] * p->dt);
      vy[i] = (float)((double)vy[i] + (double)fy[i] / (double)m[i] * p->dt);
      x[i] = (float)((double)x[i] + (double)vx[i] * p->dt);
      y[i] = (float)((double)y[i] + (double)vy[i] * p->dt);
      target[i] = NONE;
      incoming[i] = NONE;
      merged[i] = 0;
    }
    if (!p->merges) continue;
    /* S1 */
    for (uint32_t i = 0; i < n; i++) {
      sx[i] = x[i]; sy[i] = y[i]; sm[i] = alive[i] ? m[i] : 0.0f; svx[i] = vx[i]; svy[i] = vy[i];
    }
    /* pass 3: prepare_merge */
    for (uint32_t i = 0; i < n; i++) {
      if (!alive[i]) continue;
      uint32_t best = NONE;
      double bestd = 0.0;
      for (uint32_t j = 0; j < n; j++) {
        if (j == i || sm[j] == 0.0f) continue;
        int heavier = (sm[j] > sm[i]) || (sm[j] == sm[i] && j > i);
        if (!heavier) continue;
        double dx = (double)sx[j] - (double)sx[i], dy = (double)sy[j] - (double)sy[i];
        double d2 = dx * dx + dy * dy;
        if (!(d2 < R2)) continue;
        if (best == NONE || d2 < bestd || (d2 == bestd && j < best)) { best = j; bestd = d2; }
      }
      target[i] = best;
    }
    /* pass 4: claim */
    for (uint32_t i = 0; i < n; i++)
      if (alive[i] && target[i] != NONE && i < incoming[target[i]]) incoming[target[i]] = i;
    /* pass 5: absorb */
    for (uint32_t j = 0; j < n; j++) {
      if (!alive[j] || incoming[j] == NONE || target[j] != NONE) continue;
      uint32_t i = incoming[j];
      float mj = sm[j], mi = sm[i];
      float mn = mj + mi;                                  /* fp32 add */
      double md = (double)mn;
      vx[j] = (float)(((double)mj * svx[j] + (double)mi * svx[i]) / md);
      vy[j] = (float)(((double)mj * svy[j] + (double)mi * svy[i]) / md);
      x[j] = (float)(((double)mj * sx[j] + (double)mi * sx[i]) / md);
      y[j] = (float)(((double)mj * sy[j] + (double)mi * sy[i]) / md);
      m[j] = mn;
      merged[i] = 1;
    }
    /* pass 6: delete_merged */
    for (uint32_t i = 0; i < n; i++)
      if (alive[i] && merged[i]) alive[i] = 0;
  }
  free(fx); free(fy); free(target); free(incoming); free(merged);
  free(sx); free(sy); free(sm); free(svx); free(svy);
  return 0;
}
