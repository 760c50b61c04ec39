/*
 * oracle_body.h — the per-precision body of the RDCSim oracle.
 *
 * TEST INFRASTRUCTURE ONLY. Included twice by rd_oracle.c, once with
 * T=double/SFX=f64 and once with T=float/SFX=f32 ("fp64, plus an
 * fp32 mode built from the same source with T=float"). Nothing here is shared
 * with the CUDA path (paper_1901_06535_b200/csrc); the two never include each
 * other.
 *
 * Every binary floating-point operation below is written as its own C
 * expression, compiled with -ffp-contract=off and without -ffast-math, so each
 * is one IEEE-754 round-to-nearest operation in type T (x86-64 SSE2,
 * FLT_EVAL_METHOD == 0). That is the canonical expression tree of DESIGN.md
 * reading R-8.
 */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SFX)

/* The constants of Eq. 1 in type T. Each is computed in fp64 from the decimal
 * parameter and rounded ONCE to T (readings R-4, R-5; SURVEY A-4/A-5):
 *   INV_EPS = 1/eps   (the "(1/epsilon)" factor of Eq. 1)
 *   INV_DX2 = 1/dx^2  (the five-node Laplacian's scaling)
 */
typedef struct {
  T inv_eps, f, q, du, dt, inv_dx2;
} FN(orc_consts);

static FN(orc_consts) FN(make_consts)(const orc_params* p) {
  FN(orc_consts) c;
  c.inv_eps = (T)(1.0 / p->eps);
  c.f = (T)p->f;
  c.q = (T)p->q;
  c.du = (T)p->Du;
  c.dt = (T)p->dt;
  c.inv_dx2 = (T)(1.0 / (p->dx * p->dx));
  return c;
}

/* Reaction part of du/dt and dv/dt of Eq. 1:
 *   du/dt|_reaction = (1/eps) [ u - u^2 - (f v + phi) (u - q)/(u + q) ]
 *   dv/dt           = u - v
 * Evaluated as:  r = (u - q)/(u + q);  R = (u - u*u) - ((f*v + phi) * r);
 *                du = R * INV_EPS;      dv = u - v.                        */
static T FN(reaction_u)(T u, T v, T phi, const FN(orc_consts) * c) {
  T r = (u - c->q) / (u + c->q);
  T w = c->f * v;
  w = w + phi;
  T uu = u * u;
  T R = u - uu;
  R = R - (w * r);
  return R * c->inv_eps;
}

/* Five-node Laplacian at cell (i,j) with no-flux edges
 * (BASELINE.json configs "no-flux edges"; "mirroring the edge cell
 * into the out-of-grid neighbor" = ghost value := edge cell value):
 *   L = (((N + S) + (E + W)) - 4 C) * (1/dx^2)
 * (opposite neighbours paired first: DESIGN.md reading R-2).               */
static T FN(lap_at)(int64_t H, int64_t W, const T* u, int64_t i, int64_t j,
                    const FN(orc_consts) * c) {
  int64_t in = i > 0 ? i - 1 : 0;
  int64_t is = i < H - 1 ? i + 1 : H - 1;
  int64_t jw = j > 0 ? j - 1 : 0;
  int64_t je = j < W - 1 ? j + 1 : W - 1;
  T C = u[i * W + j];
  T N = u[in * W + j];
  T S = u[is * W + j];
  T E = u[i * W + je];
  T Wv = u[i * W + jw];
  T ns = N + S;
  T ew = E + Wv;
  T sum = ns + ew;
  T four_c = (T)4 * C;
  T d = sum - four_c;
  return d * c->inv_dx2;
}

/* ---- exported single-operation entry points (used by the pin tests) ---- */

double FN(orc_reaction)(double u, double v, double phi, const orc_params* p, double* dv_out) {
  FN(orc_consts) c = FN(make_consts)(p);
  T tu = (T)u, tv = (T)v, tphi = (T)phi;
  if (dv_out) *dv_out = (double)(tu - tv);
  return (double)FN(reaction_u)(tu, tv, tphi, &c);
}

void FN(orc_laplacian)(int64_t H, int64_t W, const T* u, T* out, const orc_params* p) {
  FN(orc_consts) c = FN(make_consts)(p);
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) out[i * W + j] = FN(lap_at)(H, W, u, i, j, &c);
}

/* One forward-Euler step ("explicit forward Euler
 * integration, with timestep dt"), synchronous: every output cell reads only
 * the step-s buffers:
 *   u' = u + dt * ( (1/eps)[...] + Du * L )     v' = v + dt * (u - v)
 * evaluated as  u' = C + DT*((R*INV_EPS) + (DU*L));  v' = v + DT*(C - v).
 * With ORC_REACTION_OFF: u' = C + DT*(DU*L), v' = v (the conservation pin). */
void FN(orc_step)(int64_t H, int64_t W, const T* u, const T* v, const T* phi, T* uo, T* vo,
                  const orc_params* p, uint32_t flags) {
  FN(orc_consts) c = FN(make_consts)(p);
  const int reaction = !(flags & ORC_REACTION_OFF);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < H; ++i) {
    for (int64_t j = 0; j < W; ++j) {
      int64_t k = i * W + j;
      T C = u[k];
      T L = FN(lap_at)(H, W, u, i, j, &c);
      T diff = c.du * L;
      if (reaction) {
        T Ru = FN(reaction_u)(C, v[k], phi[k], &c);
        T rhs = Ru + diff;
        uo[k] = C + c.dt * rhs;
        T dv = C - v[k];
        vo[k] = v[k] + c.dt * dv;
      } else {
        uo[k] = C + c.dt * diff;
        vo[k] = v[k];
      }
    }
  }
}

/* Stimulus stamp ("setting the excitatory concentration (u)
 * of stimulated pixels to 1.0"; SPEC.md:76-84 clip to the grid, v and phi
 * untouched). Membership is integer arithmetic in half-cell units. */
int64_t FN(orc_stamp)(int64_t H, int64_t W, T* u, const T* phi, const orc_shape* s, double value) {
  int64_t n = 0;
  T val = (T)value;
  T mphi = (T)s->mask_phi;
  for (int64_t i = 0; i < H; ++i) {
    for (int64_t j = 0; j < W; ++j) {
      if (!orc_shape_contains(s, i, j)) continue;
      if ((s->flags & ORC_SHAPE_MASK_PHI) && !(phi[i * W + j] == mphi)) continue;
      u[i * W + j] = val;
      ++n;
    }
  }
  return n;
}

/* Max of u over the rectangle [y0,y1) x [x0,x1) (SPEC.md:243-247 detect_wave:
 * "true iff max of u over the rectangle >= threshold"). NaN cells never
 * compare greater, so a NaN-only rect returns -inf. */
double FN(orc_probe_max)(int64_t H, int64_t W, const T* u, const orc_rect* r) {
  (void)H;
  T m = -(T)INFINITY;
  for (int64_t i = r->y0; i < r->y1; ++i)
    for (int64_t j = r->x0; j < r->x1; ++j)
      if (u[i * W + j] > m) m = u[i * W + j];
  return (double)m;
}

/* The whole run loop for one instance (SPEC.md:67-75 run; :438 events apply
 * before the step they are stamped with; :255, :269-270 latched detectors
 * sampled every `stride` steps; :62 abort on the first non-finite cell).
 *   for s = step0 .. step0+n-1:
 *     apply every event with at_step == s, in submission order   (a1)
 *     (u,v) <- step(u,v)                                         (a2-a5)
 *     if any non-finite cell: report first (row-major) cell, stop (a6)
 *     if (s+1) % stride == 0: latch probes with max u >= thr      (a6)
 *     if (s+1) % tl_stride == 0: timelapse max_u := max(max_u, u) (f2)
 * u, v hold the state on return (at the failing step on error). */
/* Quiescent initial state: u = v = u*(phi) of
 * each cell, computed in fp64 from the cell's phi (as stored in T) and rounded
 * once to T. */
void FN(orc_rest_fill)(int64_t H, int64_t W, const T* phi, T* u, T* v, const orc_params* p) {
  for (int64_t k = 0; k < H * W; ++k) {
    T us = (T)orc_rest_state((double)phi[k], p);
    u[k] = us;
    v[k] = us;
  }
}

/* Timelapse record ("records a timelapse ... only the concentration
 * of u is recorded over time"; SPEC.md:306-309 timelapse_record: max_u :=
 * pointwise max(max_u, u)). A NaN u never replaces the recorded value. */
void FN(orc_timelapse_record)(int64_t H, int64_t W, const T* u, T* max_u) {
  for (int64_t k = 0; k < H * W; ++k)
    if (u[k] > max_u[k]) max_u[k] = u[k];
}

int FN(orc_run)(int64_t H, int64_t W, T* u, T* v, const T* phi, const orc_params* p,
                uint32_t flags, int64_t step0, int64_t n_steps, const orc_event* events,
                int64_t n_events, const orc_probe* probes, int64_t n_probes,
                int64_t* first_fire, orc_fault* fault, int64_t tl_stride, T* tl_max) {
  T* u2 = (T*)malloc(sizeof(T) * (size_t)(H * W));
  T* v2 = (T*)malloc(sizeof(T) * (size_t)(H * W));
  if (!u2 || !v2) {
    free(u2);
    free(v2);
    return ORC_ENOMEM;
  }
  int status = ORC_OK;
  for (int64_t s = step0; s < step0 + n_steps; ++s) {
    for (int64_t e = 0; e < n_events; ++e)
      if (events[e].at_step == s) FN(orc_stamp)(H, W, u, phi, &events[e].shape, events[e].value);
    FN(orc_step)(H, W, u, v, phi, u2, v2, p, flags);
    memcpy(u, u2, sizeof(T) * (size_t)(H * W));
    memcpy(v, v2, sizeof(T) * (size_t)(H * W));
    int64_t bad = -1;
    for (int64_t k = 0; k < H * W; ++k)
      if (!isfinite(u[k]) || !isfinite(v[k])) {
        bad = k;
        break;
      }
    if (bad >= 0) {
      if (fault) {
        fault->step = s + 1;
        fault->i = bad / W;
        fault->j = bad % W;
      }
      status = ORC_ENONFINITE;
      break;
    }
    if (tl_max && tl_stride > 0 && (s + 1) % tl_stride == 0) FN(orc_timelapse_record)(H, W, u, tl_max);
    for (int64_t pi = 0; pi < n_probes; ++pi) {
      const orc_probe* pr = &probes[pi];
      if (pr->stride > 0 && (s + 1) % pr->stride == 0 && first_fire[pi] < 0) {
        double m = FN(orc_probe_max)(H, W, u, &pr->rect);
        if (m >= (double)(T)pr->threshold) first_fire[pi] = s + 1;
      }
    }
  }
  free(u2);
  free(v2);
  return status;
}

#undef FN
#undef CAT
#undef CAT2
