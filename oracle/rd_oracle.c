/*
 * rd_oracle.c — plain, slow, obviously correct CPU oracle (see rd_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline and --impl reference). Build:
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared
 * No -march flags: x86-64 SSE2 scalar arithmetic, no FTZ/DAZ.
 */
#include "rd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Table 1. phi is per cell (an input plane), not here. */
void orc_params_default(orc_params* p) {
  p->eps = 0.0243;
  p->f = 1.4;
  p->q = 0.002;
  p->Du = 0.45;
  p->dt = 0.001;
  p->dx = 0.25;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Shape membership, integer only ("every grid pixel within
 * Euclidean distance radius of center"; half-cell centres allow the exact
 * grid centre (63.5, 63.5) of an even grid, R-14). */
int orc_shape_contains(const orc_shape* s, int64_t i, int64_t j) {
  if (s->kind == ORC_RECT) return i >= s->y0 && i < s->y1 && j >= s->x0 && j < s->x1;
  int64_t dy = 2 * i - s->cy2;
  int64_t dx = 2 * j - s->cx2;
  if (dy * dy + dx * dx > 4 * s->r * s->r) return 0;
  if (s->kind == ORC_DISC) return 1;
  if (s->kind == ORC_HALF_DISC) {
    static const int64_t DX[4] = {1, 0, -1, 0};
    static const int64_t DY[4] = {0, 1, 0, -1};
    int d = s->dir & 3;
    return dx * DX[d] + dy * DY[d] >= 0;
  }
  return 0;
}

/* Homogeneous rest state (SPEC.md:85-93 steady_state: "v* = u* ... found by
 * bisection on u in (0, 1); the smallest positive root"). With v = u the
 * reaction of Eq. 1 vanishes where
 *   F(u) = (u - u*u) - ((f*u + phi) * ((u - q)/(u + q))) = 0,
 * F(0+) = phi > 0 and F(1) < 0, and the cubic it reduces to has exactly one
 * positive root. Bisection in fp64 until the midpoint no longer splits the
 * interval; returns lo (F(lo) > 0 >= F(hi), hi = next double after lo). */
double orc_rest_state(double phi, const orc_params* p) {
  const double f = p->f, q = p->q;
  double lo = 0.0, hi = 1.0;
  for (;;) {
    double mid = (lo + hi) * 0.5;
    if (!(mid > lo && mid < hi)) break;
    double r = (mid - q) / (mid + q);
    double w = f * mid;
    w = w + phi;
    double uu = mid * mid;
    double F = mid - uu;
    F = F - (w * r);
    if (F > 0.0)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

#define T double
#define SFX f64
#include "oracle_body.h"
#undef T
#undef SFX

#define T float
#define SFX f32
#include "oracle_body.h"
#undef T
#undef SFX
